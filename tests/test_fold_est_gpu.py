"""fold_est.cuh's CTA folds (cta_fold_est / cta_fold_est_rec) bit-identical to the one-thread
sequential fold (sum_residuals and best_split's boundary recording, costmodel.cpp:36-69) on
adversarial chains: builds tools/fold_bench.cu with nvcc for the CTA shapes the trainer uses
(256 threads x 16-element sub-blocks: leaves; 1,024 threads x 8: exact_small) and two others,
and runs it."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.gpu
@pytest.mark.parametrize("threads,em", [(256, 16), (1024, 8), (1024, 2), (512, 16)])
def test_fold_est_bit_exact(tmp_path, threads, em):
    exe = tmp_path / f"fold_bench_{threads}_{em}"
    subprocess.run(
        [NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false",
         f"-DLB={threads}", f"-DEM={em}", "-I", os.path.join(ROOT, "paper_2201_00194_b200", "csrc"),
         "-I", os.path.join(ROOT, "include"), "-o", str(exe), os.path.join(ROOT, "tools", "fold_bench.cu")],
        check=True, timeout=600)
    r = subprocess.run([str(exe), str(threads)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bad 0 bad_rec 0" in r.stdout
