"""Attribute ncu SASS-page metrics (stall samples, executed instructions) to
source lines: joins `ncu -i X --page source --csv --print-source sass` with
`nvdisasm -g -c <cubin>` of the same kernel (instruction offsets).

    python scripts/sass_lines.py <sass.csv> <nvdisasm.txt> <mangled-kernel> [top]
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    csvf, dis, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(csvf)))
    hdr = rows[1]
    data = rows[2:]
    ia = hdr.index("Address")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    iex = hdr.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = int(data[0][ia], 16)
    # offset -> (file, line)
    off2line = {}
    cur = None
    inside = False
    for ln in open(dis):
        if ln.startswith(".text."):
            inside = ln.strip().rstrip(":") == ".text." + fn
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m:
            off2line[int(m.group(1), 16)] = (cur, m.group(2).strip())
    agg = defaultdict(lambda: [0, 0, defaultdict(int), defaultdict(int)])
    tot = 0
    for r in data:
        off = int(r[ia], 16) - base
        key, ins = off2line.get(off, (("?", 0), "?"))
        s = int(r[isamp] or 0)
        a = agg[key]
        a[0] += s
        a[1] += int(r[iex] or 0)
        op = ins.split()[0] if ins else "?"
        if op.startswith("@"):
            op = ins.split()[1]
        a[3][op.split(".")[0]] += int(r[iex] or 0)
        for i in stall_cols:
            v = int(r[i] or 0)
            if v:
                a[2][hdr[i][6:]] += v
        tot += s
    print(f"total samples {tot}")
    for key, (s, ex, st, ops) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        sts = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4])
        opss = ", ".join(f"{k} {v//1000}k" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:4])
        print(f"{key[0]}:{key[1]:5d} {100*s/tot:5.1f}%  inst {ex/1e6:7.1f}M  [{sts}]  ({opss})")


if __name__ == "__main__":
    main()
