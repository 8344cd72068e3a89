"""Per-move instruction and stall-sample totals of the warp TabuCol kernel by
code region (source markers), from an ncu `--page source --csv --print-source
cuda,sass` export.   python tools/ncu_regions.py x.csv MOVES"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
moves = float(sys.argv[2])
src = open("paper_2109_05948_b200/csrc/tabucol_warp.cu").read().splitlines()


def find(pat):
    for i, l in enumerate(src):
        if pat in l:
            return i + 1
    return None


marks = [("expire", "// ---- tabu expiry"), ("scan1", "// ---- scan, phase 1"),
         ("phase2", "// ---- phase 2a: tie counts"), ("walks", "one walk pass over up to"), ("walks", "// ---- phase 2b: rows that lower"), ("draws", "// tenure draw (:363-365)"),
         ("locate", "// ---- locate the sstar-th"), ("move", "// ---- move, tenure, tabu entry"),
         ("update", "// ---- gamma update over N(v)"), ("events", "// events in ascending vertex order"),
         ("best", "// ---- best (:387-390)"), ("tail", "// ---- scratch check every 1024"),
         ("end", "// ---------------- outputs")]
marks = [(n, find(p)) for n, p in marks]
marks = [(n, l) for n, l in marks if l is not None]
hl = [("walk_words", "int walk_words("), ("cand_word", "__device__ __forceinline__ uint32_t cand_word"),
      ("row_min", "__device__ __forceinline__ int row_min("), ("row_count", "__device__ __forceinline__ int row_count("),
      ("count_eq", "__device__ __forceinline__ uint32_t zero_flags")]
hl = sorted([(find(p), n) for n, p in hl if find(p) is not None])
kern = find("template <int KV, int CH, bool BITSET>")


def region(f, l):
    if f != "tabucol_warp.cu":
        return "lib:" + f
    if l < kern:
        r = "helpers"
        for ln, n in hl:
            if l >= ln:
                r = n
        return r
    r = "init"
    for n, ln in marks:
        if l >= ln:
            r = n
    return r


hdr = fname = None
ins = collections.Counter()
smp = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "":
        continue
    try:
        l = int(r[0])
        i = int(r[hdr.index("Instructions Executed")])
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    g = region(fname, l)
    ins[g] += i
    smp[g] += s
ti, ts = sum(ins.values()), sum(smp.values())
print(f"total {ti / moves:.0f} warp-instructions per move")
for g, v in ins.most_common():
    print(f"{g:24s} {v / moves:8.1f} instr/move {100 * v / ti:5.1f}%i {100 * smp[g] / ts:5.1f}%samples")
