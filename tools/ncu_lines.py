"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export by
CUDA source line: warp-level instructions executed and stall samples.
    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        ins = int(r[hdr.index("Instructions Executed")])
        smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    out.append((ins, smp, f"{fname}:{r[0]}", r[1][:90]))
tot_i = sum(o[0] for o in out) or 1
tot_s = sum(o[1] for o in out) or 1
print(f"total warp instructions {tot_i:.3e}, samples {tot_s}")
for ins, smp, loc, src in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"{100*ins/tot_i:6.2f}%i {100*smp/tot_s:6.2f}%s  {loc:24s} {src}")
