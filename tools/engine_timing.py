"""Wall time of the tuning loop (TuningEngine::run, scheduler.cpp:240-290) through the three
engine builds of oracle/Makefile on one model/budget: engine_ref (the reference's own CPU cost
model), engine_b200 (the unchanged scheduler on the link-level drop-in: one device predict per
candidate) and engine_b200_batched (famtune::gpu::BatchedTuningEngine: one fs_score per pool,
fs_store append + refit per batch). Checks the three outputs are byte-identical and prints one
JSON line. Usage: python tools/engine_timing.py [model] [budget] [seed] [trees]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def run(exe, args):
    r = subprocess.run([os.path.join(REF, exe), *args], capture_output=True, text=True, timeout=3600)
    if r.returncode:
        raise SystemExit(f"{exe}: {r.stderr[-2000:]}")
    wall = [float(ln.split()[1]) for ln in r.stderr.splitlines() if ln.startswith("engine_wall_s")][0]
    return r.stdout, wall


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "mobilenetv2_sim"
    budget = sys.argv[2] if len(sys.argv) > 2 else "4000"
    seed = sys.argv[3] if len(sys.argv) > 3 else "1"
    trees = sys.argv[4] if len(sys.argv) > 4 else "50"
    args = [os.path.join(ROOT, "data", "models", model + ".json"), budget, seed, "0", "1", trees]
    out = {}
    ref_out = None
    for exe in ("engine_ref", "engine_b200", "engine_b200_batched"):
        o, w = run(exe, args)
        ref_out = ref_out or o
        out[exe] = {"wall_s": round(w, 4), "identical_to_ref": o == ref_out}
    out["config"] = {"model": model, "budget": int(budget), "seed": int(seed), "trees": int(trees),
                     "policy": "foresee, core-op families", "pool": "512 random + 512 evolved"}
    out["speedup_batched_vs_ref"] = round(out["engine_ref"]["wall_s"] / out["engine_b200_batched"]["wall_s"], 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
