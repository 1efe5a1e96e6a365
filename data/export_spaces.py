"""Export each model file as the reference LOADER sees it (after dedup and canonical reordering,
graph.cpp:265-310) into data/spaces/<name>.json: per subgraph its op-kind sequence, core op,
weight and knob value lists, plus the reference's family assignment under all three clustering
algorithms (family.cpp:105-136). These files are the inputs bench.py and the GPU tests use on
the GPU box, where /root/reference does not exist.

Usage (needs oracle/_ref, i.e. /root/reference, so run it in the build container):
    python data/export_spaces.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402  (test infrastructure; generates committed data)

MODELS = {
    "tiny": "/root/reference/proj/models/tiny.json",
    "resnet50_sim": "/root/reference/proj/models/resnet50_sim.json",
    "bert_large_sim": "/root/reference/proj/models/bert_large_sim.json",
    "mobilenetv2_sim": os.path.join(HERE, "models", "mobilenetv2_sim.json"),
    "bert_base_sim": os.path.join(HERE, "models", "bert_base_sim.json"),
}


def export(name, path):
    r = oracle.ref()
    n, pad = r.model_info(path)
    fams = {}
    csvs = {}
    for algo, tag in enumerate(("core-op", "op-count", "op-sequence")):
        f, csv = r.cluster(path, algo)
        fams[tag] = [int(v) for v in f]
        csvs[tag] = csv
    subs = []
    for s in range(n):
        info = r.subgraph_info(path, s)
        subs.append({"id": s, "ops": info["ops"], "core_op": info["core_op"], "weight": info["weight"],
                     "knobs": r.subgraph_space(path, s)})
    doc = {"name": name, "pad_dim": pad, "subgraphs": subs, "reference_families": fams,
           "reference_family_csv": csvs}
    out = os.path.join(HERE, "spaces", name + ".json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")
    print(name, n, "subgraphs, pad", pad)


if __name__ == "__main__":
    for k, v in MODELS.items():
        export(k, v)
