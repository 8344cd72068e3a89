"""Per-source-line warp instructions and stall samples (with the top stall
reasons) from an `ncu --page source --csv --print-source cuda,sass` export.
    python tools/ncu_stalls.py source.csv [moves] [top] [file-filter]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
moves = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
filt = sys.argv[4] if len(sys.argv) > 4 else ""
REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_drain", "stall_lg", "stall_long_sb",
           "stall_math", "stall_membar", "stall_mio", "stall_misc", "stall_no_inst", "stall_not_selected",
           "stall_selected", "stall_short_sb", "stall_sleep", "stall_tex", "stall_wait"]
hdr, fname, per = None, None, []
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
        st = {k: int(r[hdr.index(k)]) for k in REASONS}
    except (ValueError, IndexError):
        continue
    per.append((sum(st.values()), ins, fname, int(r[0]), r[1][:75], st))
T = sum(p[0] for p in per) or 1
I = sum(p[1] for p in per) or 1
tot = collections.Counter()
for p in per:
    tot.update(p[5])
print(f"warp instructions {I:.3e} ({I / moves:.0f} per move), stall samples {T}")
print("reasons:", {k[6:]: round(100 * v / T, 1) for k, v in tot.most_common(8)})
for s, ins, f, ln, src, st in sorted(per, key=lambda x: -x[0]):
    if filt and filt not in f:
        continue
    if top <= 0:
        break
    top -= 1
    rs = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / T:5.2f}%s {ins / moves:7.1f}i/mv {f}:{ln:<5d} {src:75s} "
          + " ".join(f"{k[6:]}={100 * v / T:.1f}" for k, v in rs if v))
