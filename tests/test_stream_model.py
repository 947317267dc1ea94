"""CPU check of the streaming (lane = row) row-pass model against brute force."""
import random

import pytest

from row_model import brute
from stream_model import expand, stream_row


@pytest.mark.parametrize("seed", range(5))
def test_stream_model_matches_bruteforce(seed):
    rnd = random.Random(seed)
    worst = 0
    for _ in range(400):
        W = rnd.randint(1, 200)
        dens = rnd.choice([0.0, 0.01, 0.05, 0.2, 0.5, 1.0])
        H = rnd.randint(1, 300)
        g = [rnd.randint(0, H) ** 2 if rnd.random() < dens else None for _ in range(W)]
        for tn in (False, True):
            want = brute(g, tn)
            for cap in (None, 4, 1):
                runs, live = stream_row(g, tn, emit_cap=cap)
                worst = max(worst, live)
                assert expand(runs, g, W) == want, (W, tn, cap, g)


def test_stream_model_ties():
    for W in (5, 17, 64):
        for step in (1, 2, 4):
            g = [0 if j % step == 0 else None for j in range(W)]
            for tn in (False, True):
                runs, _ = stream_row(g, tn)
                assert expand(runs, g, W) == brute(g, tn)
    g = [9, None, None, None, None, None, 9]  # equal parabolas, tie in the middle
    for tn in (False, True):
        runs, _ = stream_row(g, tn)
        assert expand(runs, g, 7) == brute(g, tn)


@pytest.mark.parametrize("seed", range(4))
def test_chunked_stream_model_matches_bruteforce(seed):
    """Chunks with a warm-up prefix + verification + full-prefix retry are exact
    for every chunk size / warm-up, including rows whose features all lie left
    of a chunk's warm-up (featureless-looking windows must fail verification)."""
    from stream_model import chunked_row
    rnd = random.Random(100 + seed)
    retried = 0
    for _ in range(300):
        W = rnd.randint(1, 300)
        dens = rnd.choice([0.0, 0.005, 0.02, 0.1, 0.5, 1.0])
        H = rnd.randint(1, 400)
        g = [rnd.randint(0, H) ** 2 if rnd.random() < dens else None for _ in range(W)]
        for tn in (False, True):
            want = brute(g, tn)
            for C, w in ((32, 0), (32, 32), (64, 32), (96, 64), (1000, 0)):
                got, r = chunked_row(g, C, w, tn)
                retried += r
                assert got == want, (W, tn, C, w, g)
    assert retried > 0  # the retry path is exercised
