"""bench.py's host-side contract on CPU: `--gpus N` without a launcher re-executes itself under
torchrun with N ranks (exercised through the reference arm, which needs no GPU: rank 0 alone runs
and prints one JSON line), the family partition of one global workload covers every family
exactly once, and both arms describe the workload with the same config dict."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import bench
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference (oracle/_ref) not built")
def test_gpus_flag_self_launches_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "3", "--config", "c1"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"] == bench.workload_config(bench.build_workload("c1", seed=1000))
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"


@pytest.mark.parametrize("cfg,world", [("c2", 2), ("c2", 8), ("c5", 8), ("c3", 3)])
def test_family_partition_covers_every_family_once(cfg, world):
    W = bench.build_workload(cfg, seed=1000)
    F = len(W["families"])
    seen = []
    for r in range(world):
        S = bench.shard_workload(W, r, world)
        seen += S["family_ids"]
        # the rank's rows are exactly its families' rows, in family order
        for i, f in enumerate(S["family_ids"]):
            a, b = int(W["tr_seg"][f]), int(W["tr_seg"][f + 1])
            sa, sb = int(S["tr_seg"][i]), int(S["tr_seg"][i + 1])
            assert np.array_equal(S["tr_a"][sa:sb], W["tr_a"][a:b])
            assert np.array_equal(S["tr_y"][sa:sb], W["tr_y"][a:b])
            pa, pb = int(W["pool_seg"][f]), int(W["pool_seg"][f + 1])
            qa, qb = int(S["pool_seg"][i]), int(S["pool_seg"][i + 1])
            assert np.array_equal(S["pool_a"][qa:qb], W["pool_a"][pa:pb])
        assert S["P_global"] == int(W["pool_seg"][-1]) and S["N_global"] == int(W["tr_seg"][-1])
    assert sorted(seen) == list(range(F))


def test_s8d_fit_bytes_matches_survey_formula():
    # N*D*8 + T*depth*(N*D*s_bin + 9N) + T*24N; C2's resident fit is ~240.5 MB
    W = bench.build_workload("c2", seed=1000)
    rows = [int(W["tr_seg"][f + 1] - W["tr_seg"][f]) for f in range(len(W["families"]))]
    total = sum(bench.s8d_fit_bytes(n, 100) for n in rows)
    n = sum(rows)
    assert total == n * 164 * 8 + 100 * 3 * (n * 164 + 9 * n) + 100 * 24 * n
    assert 239e6 < total < 242e6
