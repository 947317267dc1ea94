"""CPU fuzz of tests/lr_model.py -- the statement-level model of the lane-per-row
chunk scan (csrc/k_rows_lr.cu) -- against brute force, both tie rules."""
import random

import pytest

import lr_model
from row_model import brute


@pytest.mark.parametrize("take_new", [False, True])
def test_lr_model_matches_brute_force(take_new):
    rnd = random.Random(7 + take_new)
    for _ in range(1500):
        W = rnd.randint(1, 70)
        dens = rnd.choice([0.0, 0.02, 0.1, 0.5, 1.0])
        g = [(rnd.randint(0, 30) ** 2 if rnd.random() < dens else None) for _ in range(W)]
        C = rnd.randint(1, 40)
        D, K = lr_model.lr_row(g, C, take_new)
        want = brute(g, take_new)
        assert D == [w[0] for w in want] and K == [w[1] for w in want], (g, C)


@pytest.mark.parametrize("take_new", [False, True])
def test_boundary_owner_is_the_tie_rule_minimiser(take_new):
    rnd = random.Random(3)
    for _ in range(500):
        W = rnd.randint(1, 60)
        g = [(rnd.randint(0, 12) ** 2 if rnd.random() < 0.3 else None) for _ in range(W)]
        b = rnd.randrange(W)
        assert lr_model.owner(g, b, take_new) == brute(g, take_new)[b][1]


def test_live_ring_stays_small_on_discs():
    """Entry-level eager finalisation keeps the live stack far below the ring
    capacity (kLrCap = 32) on a disc image's background->object plane."""
    import numpy as np
    import oracle
    import workloads
    img = workloads.discs(256, 512, 6, 5)
    v = oracle.vertical_pass(img)
    inf = np.iinfo(np.uint64).max
    worst = 0
    for i in range(0, 256, 9):
        g = [None if x == inf else int(x) for x in v[i]]
        for c0 in range(0, 512, 128):
            c1 = c0 + 128
            kS = lr_model.owner(g, c0 - 1) if c0 else 0
            kE = lr_model.owner(g, c1 - 1) if c1 < 512 else 511
            _, st = lr_model.scan_chunk(g, c0, c1, kS, kE)
            worst = max(worst, st["max_live"])
    assert worst < 32
