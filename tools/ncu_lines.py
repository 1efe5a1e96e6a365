"""Aggregate ncu per-SASS-instruction warp-stall samples (ncu -i rep --page source --csv
--print-source sass) onto CUDA source lines, using nvdisasm -g line info of the same cubin.

    python tools/ncu_lines.py SASS_CSV NVDISASM_G_OUTPUT KERNEL_SYMBOL [top]
"""
import collections
import csv
import re
import sys


def line_map(sass_path, symbol):
    amap, cur, inside = {}, None, False
    for ln in open(sass_path):
        if ln.startswith(".text.") or ln.startswith("//--------------------- .text."):
            inside = symbol in ln
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            amap[int(m.group(1), 16)] = cur
    return amap


def main():
    csv_path, sass_path, symbol = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    amap = line_map(sass_path, symbol)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = int(rows[2][ia], 16)
    per = collections.defaultdict(lambda: collections.Counter())
    total = 0
    for r in rows[2:]:
        if len(r) <= isamp:
            continue
        off = int(r[ia], 16) - base
        s = int(r[isamp] or 0)
        total += s
        key = amap.get(off, ("?", 0))
        per[key]["samples"] += s
        for i in stall_cols:
            v = int(r[i] or 0)
            if v:
                per[key][hdr[i]] += v
    print("total samples", total)
    for key, c in sorted(per.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        reasons = sorted(((k, v) for k, v in c.items() if k != "samples"), key=lambda kv: -kv[1])[:3]
        print(f"{c['samples']:7d} {100.0 * c['samples'] / max(total, 1):5.1f}%  {key[0]}:{key[1]}  " +
              " ".join(f"{k[6:]}={v}" for k, v in reasons))


if __name__ == "__main__":
    main()
