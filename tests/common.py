"""Shared, numpy-only input builders for the parity tests and bench.py-independent checks.

Model knob spaces come from data/spaces/*.json (exported from the reference loader by
data/export_spaces.py) so everything here runs on the GPU box without /root/reference.
"""
from __future__ import annotations

import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def load_spaces(name: str) -> dict:
    with open(os.path.join(ROOT, "data", "spaces", name + ".json")) as f:
        return json.load(f)


def families(doc: dict, algo: str = "core-op") -> dict[int, list[int]]:
    out: dict[int, list[int]] = {}
    for sid, fam in enumerate(doc["reference_families"][algo]):
        out.setdefault(fam, []).append(sid)
    return out


def random_assignments(rng: np.random.Generator, knobs: list[list[int]], n: int, distinct: bool = True):
    """n assignments (value indices) drawn uniformly; distinct when the space allows it."""
    sizes = [len(v) for v in knobs]
    total = int(np.prod(sizes))
    if distinct and n <= total:
        lin = rng.choice(total, size=n, replace=False)
    else:
        lin = rng.integers(0, total, size=n)
    a = np.zeros((n, 16), np.int32)
    for k in range(len(sizes) - 1, -1, -1):
        a[:, k] = lin % sizes[k]
        lin = lin // sizes[k]
    return a


def synth_latency(rng: np.random.Generator, knobs, assign, noise=0.02, seed_shift=0):
    """A quadratic bowl over normalized knob positions (the shape of simbackend.cpp:80-102),
    lognormal noise. Deterministic for a given rng state."""
    k = len(knobs)
    z = np.stack([assign[:, i] / max(len(knobs[i]) - 1, 1) for i in range(k)], axis=1)
    opt = rng.uniform(0, 1, size=k)
    curv = rng.uniform(0.5, 2.0)
    w = rng.uniform(-0.01, 0.01, size=(k, k))
    w = (w + w.T) / 2
    np.fill_diagonal(w, 0)
    base = np.exp(rng.uniform(np.log(0.1), np.log(10.0)))
    quad = curv * ((z - opt) ** 2).sum(1)
    inter = np.einsum("ni,ij,nj->n", z, w, z)
    lat = base * (1.0 + quad + inter)
    if noise:
        lat = lat * np.exp(rng.normal(0, noise, size=len(lat)))
    return lat


def family_dataset(doc, members, per_subgraph, pad_dim, seed, orc):
    """Rows for one family: random distinct candidates per member subgraph, features from the
    oracle featurize (pinned to the reference), synthetic latencies. Returns
    (x, latency, space_of, assign)."""
    rng = np.random.default_rng(seed)
    xs, ls, so, aa = [], [], [], []
    for sid in members:
        knobs = doc["subgraphs"][sid]["knobs"]
        total = int(np.prod([len(v) for v in knobs]))
        n = min(per_subgraph, total)
        a = random_assignments(rng, knobs, n)
        x = orc.featurize(knobs, a[:, : len(knobs)], pad_dim)
        lat = synth_latency(rng, knobs, a)
        xs.append(x)
        ls.append(lat)
        so.append(np.full(n, sid, np.int32))
        aa.append(a)
    return np.concatenate(xs), np.concatenate(ls), np.concatenate(so), np.concatenate(aa)


def random_dataset(seed, n, d, kind="c7"):
    """Continuous-feature datasets in the style of the reference's property tests
    (costmodel_test.cpp:185-202, acceptance_test.cpp:325-340)."""
    rng = np.random.default_rng(seed)
    if kind == "c7":
        x = np.stack([rng.uniform(0, 4, n), rng.uniform(0, 4, n), rng.uniform(0, 4, n), rng.uniform(0, 1, n)], 1)
        y = 2 * x[:, 0] - x[:, 1] * x[:, 2] + np.sin(x[:, 3]) + rng.normal(0, 0.25, n)
    elif kind == "mse":
        x = np.stack([rng.uniform(0, 8, n), rng.uniform(0, 8, n), rng.uniform(0, 1, n)], 1)
        y = x[:, 0] * 0.5 - x[:, 1] * x[:, 2] + rng.normal(0, 0.3, n)
    elif kind == "discrete":
        x = rng.integers(0, 6, size=(n, d)).astype(np.float64)
        y = x[:, 0] - 0.5 * x[:, 1 % d] + rng.normal(0, 0.1, n)
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(x), np.ascontiguousarray(y)


def spaces_list(doc):
    return [s["knobs"] for s in doc["subgraphs"]]
