"""Family grouping is bit-exact with the reference (family.cpp:22-140): ids, members and the
registry CSV under all three clustering algorithms, for every model file (the expected values in
data/spaces/*.json were produced by the reference itself, data/export_spaces.py). CPU only."""
import pytest

from common import load_spaces
from paper_2201_00194_b200 import families

MODELS = ["tiny", "resnet50_sim", "bert_large_sim", "mobilenetv2_sim", "bert_base_sim"]


@pytest.mark.parametrize("model", MODELS)
@pytest.mark.parametrize("algo", ["core-op", "op-count", "op-sequence"])
def test_matches_reference(model, algo):
    doc = load_spaces(model)
    fam, csv = families.cluster(doc["subgraphs"], algo)
    assert fam.tolist() == doc["reference_families"][algo]
    assert csv == doc["reference_family_csv"][algo]


def test_exact_csv_and_errors():
    # family_test.cpp:187-194
    fam, csv = families.cluster([{"core_op": "conv2d", "ops": ["conv2d"]},
                                 {"core_op": "softmax", "ops": ["softmax"]}])
    assert csv == "subgraph_id,family_id,signature\n0,0,conv2d\n1,1,softmax\n"
    with pytest.raises(ValueError):
        families.cluster([])


def test_permutation_invariant_partition():
    # family_test.cpp:135-170: the partition does not depend on subgraph order (ids do)
    doc = load_spaces("resnet50_sim")
    subs = doc["subgraphs"]
    fam, _ = families.cluster(subs)
    rev = list(reversed(subs))
    fam_r, _ = families.cluster(rev)
    groups = {frozenset(i for i in range(len(subs)) if fam[i] == f) for f in set(fam.tolist())}
    groups_r = {frozenset(len(subs) - 1 - i for i in range(len(rev)) if fam_r[i] == f) for f in set(fam_r.tolist())}
    assert groups == groups_r
