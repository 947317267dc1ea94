"""CPU check of the row-pass merge algorithm (tests/row_model.py mirrors
paper_2106_03503_b200/csrc/k_rows.cu statement for statement) against brute
force, for both tie rules, many segment geometries and densities."""
import random

import pytest

from row_model import brute, row_envelope


@pytest.mark.parametrize("seed", range(6))
def test_row_model_matches_bruteforce(seed):
    rnd = random.Random(seed)
    for _ in range(250):
        W = rnd.randint(1, 260)
        T = rnd.choice([1, 2, 4, 8, 16, 32, 64])
        L = 4
        while T * L < W:
            L *= 2
        dens = rnd.choice([0.0, 0.01, 0.05, 0.2, 0.5, 1.0])
        H = rnd.randint(1, 300)
        g = [rnd.randint(0, H) ** 2 if rnd.random() < dens else None for _ in range(W)]
        for take_new in (False, True):
            want = brute(g, take_new)
            assert row_envelope(g, T, L, take_new, True) == want, (W, T, L, take_new)
            assert row_envelope(g, T, L, take_new, False) == want, (W, T, L, take_new)
            assert row_envelope(g, T, L, take_new, "probe") == want, (W, T, L, take_new)


def test_row_model_ties():
    # equal parabolas everywhere: keep_old -> smallest column, take_new -> largest
    for W in (5, 17, 64):
        g = [0 if j % 4 == 0 else None for j in range(W)]
        for T in (1, 4, 16):
            L = 4
            while T * L < W:
                L *= 2
            for tn in (False, True):
                assert row_envelope(g, T, L, tn) == brute(g, tn)
