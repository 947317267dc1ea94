"""CPU fuzz of tests/anc_model.py -- the statement-level model of the anchored-
segment row pass (csrc/k_rows_anc.cu) -- against brute force, both tie rules,
segment widths 1..40, the kernel's aligned superset scan, ties and empty columns."""
import random

import pytest

import anc_model
from row_model import brute


@pytest.mark.parametrize("take_new", [False, True])
@pytest.mark.parametrize("superset", [False, True])
def test_anc_model_matches_brute_force(take_new, superset):
    rnd = random.Random(11 + 2 * take_new + superset)
    for _ in range(1500):
        W = rnd.randint(1, 90)
        dens = rnd.choice([0.0, 0.02, 0.1, 0.5, 1.0])
        hmax = rnd.choice([1, 3, 12, 30])  # small heights: many ties
        g = [(rnd.randint(0, hmax) ** 2 if rnd.random() < dens else None) for _ in range(W)]
        L = rnd.choice([1, 2, 3, 5, 8, 32, 40])
        D, K = anc_model.anc_row(g, take_new, L, superset)
        want = brute(g, take_new)
        assert D == [w[0] for w in want], (g, L)
        assert K == [w[1] for w in want], (g, L)  # owners too: a superset holds no extra minimiser
