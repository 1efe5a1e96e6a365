"""Family-parallel sharding across GPUs (one process per GPU).

Families share nothing (scheduler.cpp:123-130: one CostModelState, training set and pool each),
so they are partitioned across ranks with no data-path collective. The only exchange is the
per-round all-gather of each family's top-g candidates, merged in family-id order on every
rank. Results per family are bit-identical whichever rank computes them.
"""
from __future__ import annotations

import numpy as np

RECORD_FIELDS = 4  # family id, subgraph id, pool index, score (all carried as float64)


def family_cost(n_rows: int, n_pool: int, trees: int) -> float:
    """Cost estimate used for balancing: boosting work (rows x trees) + scoring (pool x trees)."""
    return float(n_rows) * trees + float(n_pool) * trees


def assign_families(costs, world: int) -> list[int]:
    """Deterministic LPT bin packing: families in descending cost (ties: lower id first) go to
    the least-loaded rank (ties: lower rank). Returns rank per family."""
    order = sorted(range(len(costs)), key=lambda f: (-costs[f], f))
    load = [0.0] * world
    owner = [0] * len(costs)
    for f in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[f] = r
        load[r] += costs[f]
    return owner


def pack_topk(family_ids, seg, perm, scores, g: int, subgraph_of=None) -> np.ndarray:
    """Fixed-size records [len(family_ids) * g, 4] of each family's first g ranked candidates
    (tune_step's by-score picks, scheduler.cpp:196-201); short pools are padded with family -1."""
    out = np.full((len(family_ids) * g, RECORD_FIELDS), -1.0)
    for i, fam in enumerate(family_ids):
        a, b = int(seg[i]), int(seg[i + 1])
        k = min(g, b - a)
        idx = np.asarray(perm[a:a + k], np.int64)
        rows = out[i * g: i * g + k]
        rows[:, 0] = fam
        rows[:, 1] = -1 if subgraph_of is None else np.asarray(subgraph_of[a:b])[idx]
        rows[:, 2] = idx
        rows[:, 3] = np.asarray(scores[a:b])[idx]
    return out


def merge_topk(gathered: np.ndarray, g: int) -> dict[int, np.ndarray]:
    """All-gathered records -> {family id: [k, 4] records in rank order}, families ascending."""
    recs = gathered.reshape(-1, g, RECORD_FIELDS)
    out = {}
    for block in recs:
        valid = block[block[:, 0] >= 0]
        if len(valid):
            out[int(valid[0, 0])] = valid
    return dict(sorted(out.items()))
