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
