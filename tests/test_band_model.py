"""CPU fuzz of tests/band_model.py -- the statement-level model of the
band-candidate row pass for sparse planes (csrc/k_rows_band.cu: hull filter,
lane-per-row stack with a spilling ring, fill) -- against brute force, both
tie rules, with small windows / lanes / ring capacities so that the bridge
merges, the window boundaries and the spill / reload paths all run."""
import random

import pytest

import band_model as bm


def _img(rnd, H, W, dens, mode):
    img = [[0] * W for _ in range(H)]
    if mode == "bern":
        for i in range(H):
            for j in range(W):
                img[i][j] = 1 if rnd.random() < dens else 0
    elif mode == "rowline":  # a full object row: every column on the hull
        r = rnd.randrange(H)
        img[r] = [1] * W
    elif mode == "few":
        for _ in range(rnd.randint(0, 4)):
            img[rnd.randrange(H)][rnd.randrange(W)] = 1
    elif mode == "lattice":  # many exact ties
        s = rnd.randint(2, 6)
        for i in range(rnd.randrange(s), H, s):
            for j in range(rnd.randrange(s), W, s):
                img[i][j] = 1
    return img


@pytest.mark.parametrize("take_new", [False, True])
def test_band_model_matches_brute_force(take_new):
    rnd = random.Random(11 + take_new)
    for it in range(140):
        H = rnd.randint(1, 100)
        W = rnd.randint(1, 48)
        mode = rnd.choice(["bern", "bern", "rowline", "few", "lattice"])
        img = _img(rnd, H, W, rnd.choice([0.0, 0.005, 0.02, 0.1, 0.4]), mode)
        lane_cols = rnd.choice([1, 2, 3, 4, 8, 32])
        lanes = rnd.choice([1, 2, 4, 8, 32])
        cap = rnd.choice([1, 2, 3, 32])
        hcap = rnd.choice([None, 2, 3, 5])   # hull stacks that overflow: all valid columns
        D, K, R, _, _ = bm.band_transform(img, take_new, cap, lane_cols, lanes, hcap)
        bD, bK, bR = bm.brute(img, take_new)
        assert D == bD, (it, mode, H, W)
        assert K == bK, (it, mode, H, W)
        if not take_new:
            assert R == bR, (it, mode, H, W)


def test_window_hull_is_superset_of_global_hull():
    rnd = random.Random(5)
    for _ in range(300):
        W = rnd.randint(1, 90)
        line = rnd.randint(0, 200)
        car = [rnd.randint(0, 199) if rnd.random() < 0.6 else None for _ in range(W)]
        car = [None if c is None else min(c, line) for c in car]
        glob = bm.window_hull(car, line, 0, lane_cols=W, lanes=1)
        for lc, ln in ((1, 4), (3, 4), (4, 8), (32, 32)):
            got = set()
            for w0 in range(0, W, lc * ln):
                got |= bm.window_hull(car, line, w0, lc, ln, W)
            assert glob <= got
            # one window covering the whole row: the merges give exactly the global hull
        assert bm.window_hull(car, line, 0, 1, 128, W) == glob


def test_candidate_counts_are_small_on_sparse_tiles():
    """Candidate columns per band on a scaled C5-like image stay far below W
    (the row pass's work); the spill path never runs at the kernel's cap."""
    rnd = random.Random(2)
    H, W = 96, 512
    img = [[0] * W for _ in range(H)]
    for _ in range(40):
        img[rnd.randrange(H)][rnd.randrange(W)] = 1
    _, _, _, ncand, st = bm.band_transform(img, False, 32, 32, 32)
    assert max(ncand) < W // 3
    assert st["spills"] == 0


@pytest.mark.parametrize("take_new", [False, True])
def test_band_model_grouped_chunked(take_new):
    """Grouped candidates (hulls at the group's first / last band + the
    group's object columns) and chunked stacks with exact scan bounds."""
    rnd = random.Random(23 + take_new)
    for it in range(60):
        H = rnd.randint(1, 140)
        W = rnd.randint(1, 100)
        mode = rnd.choice(["bern", "bern", "rowline", "few", "lattice"])
        img = _img(rnd, H, W, rnd.choice([0.0, 0.003, 0.02, 0.1, 0.4]), mode)
        D, K, R = bm.band_transform_chunked(img, take_new, nch=rnd.choice([1, 2, 3, 8]),
                                            cap=rnd.choice([1, 2, 16]), group=rnd.choice([1, 2, 4]))
        bD, bK, bR = bm.brute(img, take_new)
        assert D == bD, (it, mode, H, W)
        assert K == bK, (it, mode, H, W)
        if not take_new:
            assert R == bR, (it, mode, H, W)


def test_list_prune_is_superset_of_hull_and_converges():
    """warp_prune: never drops a hull point (collinear ones included), whatever
    the number of rounds; with enough rounds it reaches the hull itself."""
    rnd = random.Random(8)
    for _ in range(150):
        W = rnd.randint(1, 160)
        line = rnd.randint(0, 300)
        car = [rnd.randint(0, line) if rnd.random() < rnd.choice([0.1, 0.6, 1.0]) else None for _ in range(W)]
        r = rnd.random()
        if r < 0.15:    # equal carries on a column lattice
            car = [line - 3 if k % 2 == 0 else None for k in range(W)]
        elif r < 0.3:   # bowls between deep minima
            car = [line - rnd.randint(40, 60) for _ in range(W)]
            for _ in range(rnd.randint(1, 4)):
                car[rnd.randrange(W)] = line
        glob = bm.window_hull(car, line, 0, lane_cols=W, lanes=1)
        pts = [(k, (line - car[k]) ** 2 + k * k) for k in range(W) if car[k] is not None]
        for rounds in (0, 1, 2, 10):
            got = bm.list_prune(pts, rounds)
            assert glob <= got <= set(k for k, _ in pts)
        assert bm.list_prune(pts, 10 ** 6, strides=(1,)) == glob  # the fixed point of stride 1 is the hull


@pytest.mark.parametrize("take_new", [False, True])
def test_band_model_hierarchical_hulls(take_new):
    """Coarse lines over all columns, group lines over the coarse survivors plus
    the object columns in between (k_hull<0/1/2>, any number of prune rounds),
    then the chunked stacks: equal to brute force; and the group lines' filters
    contain the hulls over all columns."""
    rnd = random.Random(31 + take_new)
    for it in range(30):
        H = rnd.randint(1, 300)
        W = rnd.randint(1, 70)
        mode = rnd.choice(["bern", "bern", "rowline", "few", "lattice"])
        img = _img(rnd, H, W, rnd.choice([0.0, 0.003, 0.02, 0.1]), mode)
        group = rnd.choice([1, 2])
        coarse = group * rnd.choice([1, 2, 4])
        D, K, R = bm.band_transform_chunked(img, take_new, nch=rnd.choice([1, 3, 8]), cap=rnd.choice([2, 16]),
                                            group=group, coarse=coarse, lanes=rnd.choice([0, 1, 3, 10]),
                                            win=rnd.choice([None, 8, 32]), hcap=rnd.choice([None, 3, 10]))
        bD, bK, bR = bm.brute(img, take_new)
        assert D == bD, (it, mode, H, W)
        assert K == bK, (it, mode, H, W)
        if not take_new:
            assert R == bR, (it, mode, H, W)
        if it % 5 == 0:  # the hierarchy loses no hull point
            above, below, masks = bm.carries(img, H, W)
            nb = (H + 31) // 32
            for g0 in range(0, nb, group):
                g1 = min(nb - 1, g0 + group - 1)
                cb0 = g0 // coarse * coarse
                got = bm.hier_group_candidates(above, below, masks, g0, g1, cb0, min(nb - 1, cb0 + coarse - 1), H, W)
                want = set(k for bb in range(g0, g1 + 1) for k in range(W) if masks[bb][k])
                want |= bm.window_hull(above[g0], 32 * g0, 0, W, 1, W)
                want |= bm.window_hull(below[g1], min(32 * g1 + 31, H - 1), 0, W, 1, W)
                assert got >= want
