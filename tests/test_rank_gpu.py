"""GPU ranking vs std::sort over (score, index) pairs (scheduler.cpp:187-192): full permutation,
bit-exact, including ties, signed zeros and segments that span several sort chunks."""
import numpy as np
import pytest

import paper_2201_00194_b200 as fs
from common import GOLDEN

pytestmark = pytest.mark.gpu
G = np.load(f"{GOLDEN}/golden.npz")


def test_golden_ties_and_signed_zeros(dev):
    assert np.array_equal(dev.rank(G["rank_scores"]), G["rank_perm"])


@pytest.mark.parametrize("sizes", [[1], [2, 0, 3], [4096], [4097], [8192, 12000, 5], [65536], [100000, 17, 70000]])
def test_segments(dev, orc, sizes):
    rng = np.random.default_rng(sum(sizes))
    n = sum(sizes)
    s = np.round(rng.normal(0, 1, n), 3)  # many exact ties
    s[rng.random(n) < 0.05] = -0.0
    seg = np.concatenate([[0], np.cumsum(sizes)])
    perm = dev.rank(s, seg)
    for i in range(len(sizes)):
        a, b = seg[i], seg[i + 1]
        assert np.array_equal(perm[a:b], orc.rank(s[a:b])), i


def test_extremes(dev, orc):
    s = np.array([np.inf, -np.inf, 1e308, -1e308, 5e-324, -5e-324, 0.0, -0.0, 1.0, 1.0])
    assert np.array_equal(dev.rank(s), orc.rank(s))
