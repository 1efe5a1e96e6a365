"""Batched pairwise accuracy (costmodel.cpp:248-277; the accuracy heatmap's model x
validation-set grid, experiment.cpp:135-167) vs the oracle, segment by segment."""
import numpy as np
import pytest

import paper_2201_00194_b200 as fs

pytestmark = pytest.mark.gpu


def test_batch_matches_single_and_oracle(dev, orc):
    rng = np.random.default_rng(5)
    sizes = [2, 7, 64, 300, 1000]
    seg = np.concatenate([[0], np.cumsum(sizes)])
    lat = np.exp(rng.normal(0, 1, seg[-1]))
    lat[10:14] = lat[10]  # latency ties (excluded pairs)
    scores = np.log(lat) + rng.normal(0, 0.3, seg[-1])
    scores[70:90] = 0.25  # predicted ties (half credit)
    got = dev.pairwise_accuracy_batch(scores, lat, seg)
    for k in range(len(sizes)):
        a, b = seg[k], seg[k + 1]
        exp = orc.pairwise_accuracy(scores[a:b], lat[a:b])
        assert got[k] == exp
        assert dev.pairwise_accuracy(scores[a:b], lat[a:b]) == exp


def test_batch_errors(dev):
    with pytest.raises(fs.InvalidArgument):
        dev.pairwise_accuracy_batch(np.zeros(3), np.ones(3), [0, 2, 3])  # a 1-record segment
    with pytest.raises(fs.DomainError):
        dev.pairwise_accuracy_batch(np.zeros(4), np.ones(4), [0, 2, 4])  # every pair a latency tie
