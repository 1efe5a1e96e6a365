"""Bucket ncu per-SASS warp-stall samples of the resident trainer by phase: a phase is the span
of fit_resident.cuh lines after each '// ---- <name>' marker comment. Barrier stalls and the
rest are reported separately (barrier samples sit at the barrier that ENDS a phase).

    python tools/ncu_phases.py SASS_CSV NVDISASM_G_OUTPUT KERNEL_SYMBOL SOURCE_FILE
"""
import collections
import csv
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_lines import line_map  # noqa: E402


def main():
    csv_path, sass_path, symbol, src_path = sys.argv[1:5]
    amap = line_map(sass_path, symbol)
    marks = []
    for no, ln in enumerate(open(src_path), 1):
        m = re.match(r"\s*// ---- ([a-zA-Z][^(\-:]*)", ln)
        if m:
            marks.append((no, m.group(1).strip()[:28]))
    fname = src_path.rsplit("/", 1)[-1]

    def phase(f, l):
        if f != fname:
            return "other:" + f
        name = "prologue"
        for no, nm in marks:
            if no <= l:
                name = nm
        return name

    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ia = hdr.index("Address")
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    ib = hdr.index("stall_barrier")
    base = int(rows[2][ia], 16)
    work, bar = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= max(cols):
            continue
        f, l = amap.get(int(r[ia], 16) - base, ("?", 0))
        p = phase(f, l)
        bar[p] += int(r[ib] or 0)
        work[p] += sum(int(r[i] or 0) for i in cols if i != ib)
    tw, tb = sum(work.values()), sum(bar.values())
    print(f"non-barrier samples {tw}, barrier samples {tb}")
    for p, v in work.most_common():
        print(f"{p:30s} work {v:6d} {100 * v / tw:5.1f}%   barrier {bar[p]:6d}")


if __name__ == "__main__":
    main()
