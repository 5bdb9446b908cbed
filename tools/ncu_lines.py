"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass -k regex:K > x.csv; python tools/ncu_lines.py x.csv [kernel-substr] [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
fname, func, hdr = None, None, None
agg = collections.defaultdict(lambda: collections.Counter())
srcs = {}
tot = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or want not in (func or ""):
        continue
    if r[0] and r[0] != "":
        key = (fname, int(r[0]))
        srcs[key] = r[1][:70]
        def g(c):
            try:
                return int(float(r[hdr[c]]))
            except (KeyError, ValueError):
                return 0
        s = g("Warp Stall Sampling (All Samples)")
        agg[key]["samples"] += s
        agg[key]["inst"] += g("Instructions Executed")
        for c in hdr:
            if c.startswith("stall_") and "Not Issued" not in c:
                agg[key][c] += g(c)
        tot["samples"] += s
        tot["inst"] += g("Instructions Executed")
print("total samples", tot["samples"], "warp-instructions", tot["inst"])
for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = sorted(((k[6:], v) for k, v in c.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:3]
    print(f"{c['samples'] / tot['samples'] * 100:5.1f}% inst {c['inst'] / tot['inst'] * 100:5.1f}%  {key[0]}:{key[1]:<4} "
          f"{srcs[key]:<70} {' '.join(f'{k}={v / max(c[chr(115)+chr(97)+chr(109)+chr(112)+chr(108)+chr(101)+chr(115)], 1):.2f}' for k, v in st)}")
