"""End-to-end drop-in gate: the reference's UNCHANGED tuning engine
(scheduler.cpp, simbackend.cpp, ...) linked against libfamtune_b200.so instead of its own
costmodel.cpp / family.cpp must produce a byte-identical convergence curve, family registry and
per-family model digests (mirrors scheduler_test.cpp:300-308's deterministic-curve check, but
across implementations). The batched caller (famtune::gpu::BatchedTuningEngine: one fs_score per
pool, fs_store append + refit per measured batch) must produce the same bytes too. Also runs the
drop-in C++ API test program."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
ENG_REF = os.path.join(REF, "engine_ref")
ENG_B200 = os.path.join(REF, "engine_b200")
ENG_BATCHED = os.path.join(REF, "engine_b200_batched")
API_TEST = os.path.join(ROOT, "tests", "cpp", "famtune_api_test")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(API_TEST), reason="tests/cpp/famtune_api_test not built")
def test_cpp_dropin_api():
    r = subprocess.run([API_TEST], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.skipif(not (os.path.exists(ENG_REF) and os.path.exists(ENG_B200)), reason="engines not built")
@pytest.mark.parametrize("model,budget,seed,algo,foresee,trees", [
    ("bert_base_sim", 300, 1, 0, 1, 50),
    ("bert_base_sim", 400, 7, 2, 1, 30),
    ("mobilenetv2_sim", 500, 3, 0, 1, 50),
    ("mobilenetv2_sim", 400, 5, 1, 0, 40),
])
def test_engine_curve_identical(model, budget, seed, algo, foresee, trees):
    path = os.path.join(ROOT, "data", "models", model + ".json")
    args = [path, str(budget), str(seed), str(algo), str(foresee), str(trees)]
    a = subprocess.run([ENG_REF, *args], capture_output=True, text=True, timeout=600)
    b = subprocess.run([ENG_B200, *args], capture_output=True, text=True, timeout=600)
    assert a.returncode == 0, a.stderr
    assert b.returncode == 0, b.stderr
    assert "model family=" in a.stdout
    assert a.stdout == b.stdout
    if os.path.exists(ENG_BATCHED):
        c = subprocess.run([ENG_BATCHED, *args], capture_output=True, text=True, timeout=600)
        assert c.returncode == 0, c.stderr
        assert a.stdout == c.stdout


@pytest.mark.skipif(not (os.path.exists(ENG_REF) and os.path.exists(ENG_BATCHED)), reason="engines not built")
@pytest.mark.parametrize("model,budget,seed,algo,foresee,trees", [
    ("mobilenetv2_sim", 1500, 2, 0, 1, 50),  # core-op families, foresee phase
    ("bert_base_sim", 900, 4, 0, 0, 50),     # monolithic baseline: one model for every subgraph
])
def test_batched_engine_identical(model, budget, seed, algo, foresee, trees):
    path = os.path.join(ROOT, "data", "models", model + ".json")
    args = [path, str(budget), str(seed), str(algo), str(foresee), str(trees)]
    a = subprocess.run([ENG_REF, *args], capture_output=True, text=True, timeout=900)
    c = subprocess.run([ENG_BATCHED, *args], capture_output=True, text=True, timeout=900)
    assert a.returncode == 0, a.stderr
    assert c.returncode == 0, c.stderr
    assert "model family=" in a.stdout
    assert a.stdout == c.stdout
