"""Generate tests/golden/linear_index.npz: the UNMODIFIED reference's linear_index and
candidate_from_index (searchspace.cpp:48-66, via oracle/_ref) on every subgraph space of the
resnet50_sim and bert_base_sim model files, 64 random assignments per space (seed 7) plus each
space's first and last assignment. Runs where /root/reference exists:
    python tests/golden/make_golden_index.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from common import load_spaces, random_assignments, spaces_list  # noqa: E402


def main():
    ref = oracle.ref()
    rng = np.random.default_rng(7)
    out = {}
    for name in ("resnet50_sim", "bert_base_sim"):
        for sid, knobs in enumerate(spaces_list(load_spaces(name))):
            a = random_assignments(rng, knobs, 64, distinct=False)
            first = np.zeros((1, 16), np.int32)
            last = np.zeros((1, 16), np.int32)
            last[0, : len(knobs)] = [len(v) - 1 for v in knobs]
            a = np.concatenate([first, a, last])
            idx = ref.linear_index(knobs, a[:, : len(knobs)])
            back = ref.candidate_from_index(knobs, idx)
            out[f"{name}_{sid}_assign"] = a
            out[f"{name}_{sid}_index"] = idx
            out[f"{name}_{sid}_back"] = back
    np.savez_compressed(os.path.join(HERE, "linear_index.npz"), **out)
    print(len(out) // 3, "spaces")


if __name__ == "__main__":
    main()
