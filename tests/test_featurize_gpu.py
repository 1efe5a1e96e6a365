"""GPU featurize (kernel 1) vs the oracle restatement and the reference's exact-value pins
(searchspace_test.cpp:59-100). Bit-exact."""
import numpy as np
import pytest

import paper_2201_00194_b200 as fs
from common import GOLDEN, load_spaces, random_assignments, spaces_list

pytestmark = pytest.mark.gpu
G = np.load(f"{GOLDEN}/golden.npz")


def test_exact_layouts(dev):
    sp = fs.Spaces(dev, [[[8, 16, 32]], [[4, 8], [2, 16]], [[1, 2, 4, 8], [1, 3, 9], [2, 4]]])
    assert np.array_equal(sp.featurize([0], [[0]], 6)[0], G["feat_single"])
    assert np.array_equal(sp.featurize([1], [[0, 0]], 5)[0], G["feat_pair"])
    small = sp.featurize(np.full(24, 2), G["feat_small_assign"], 9)
    assert np.array_equal(small, G["feat_small"])


@pytest.mark.parametrize("name,pad", [("resnet50_sim", 164), ("bert_base_sim", 164), ("mobilenetv2_sim", 14),
                                      ("bert_base_sim", 27)])
def test_model_spaces_bitexact(dev, orc, name, pad):
    doc = load_spaces(name)
    spaces = spaces_list(doc)
    sp = fs.Spaces(dev, spaces)
    assert sp.max_feature_dim == doc["pad_dim"]
    rng = np.random.default_rng(1)
    so = rng.integers(0, len(spaces), 3000).astype(np.int32)
    asg = np.zeros((len(so), 16), np.int32)
    for i, s in enumerate(so):
        asg[i] = random_assignments(rng, spaces[s], 1, distinct=False)[0]
    got = sp.featurize(so, asg, pad)
    for s in np.unique(so):
        rows = np.where(so == s)[0]
        exp = orc.featurize(spaces[s], asg[rows, : len(spaces[s])], pad)
        assert np.array_equal(got[rows], exp), s


def test_sixteen_knob_space_pad164(dev, orc):
    rng = np.random.default_rng(2)
    knobs = [[2 ** j for j in range(int(rng.integers(4, 9)))] for _ in range(16)]
    sp = fs.Spaces(dev, [knobs])
    a = random_assignments(rng, knobs, 5000)
    got = sp.featurize(np.zeros(5000, np.int32), a, 164)
    assert np.array_equal(got, orc.featurize(knobs, a, 164))
    assert np.all(got[:, 152:] == 0.0)


def test_errors(dev):
    sp = fs.Spaces(dev, [[[1, 2], [1, 2]]])
    with pytest.raises(fs.InvalidArgument):  # searchspace.cpp:96-100
        sp.featurize([0], [[0, 0]], fs.feature_dim(2) - 1)
    with pytest.raises(fs.InvalidArgument):
        sp.featurize([0], [[0, 2]], 8)
    with pytest.raises(fs.InvalidArgument):
        sp.featurize([1], [[0, 0]], 8)
    with pytest.raises(fs.InvalidArgument):
        fs.Spaces(dev, [[[0, 1]]])  # non-positive value (validate_space)
    # device stays usable after deferred errors
    assert np.array_equal(sp.featurize([0], [[1, 1]], 5)[0], [1.0, 1.0, 1.0, 1.0, 1.0])
