"""Static SASS instruction count of one warp-kernel instantiation by code
region (hot-loop code size; the instruction cache is a first-order limit).
    python tools/sass_regions.py <object.o> [instantiation-substring]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj = sys.argv[1]
inst = sys.argv[2] if len(sys.argv) > 2 else "ILi3ELi16ELb1"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(os.path.join(root, "paper_2109_05948_b200/csrc/tabucol_warp.cu")).read().splitlines()
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(td, cub)], capture_output=True, text=True).stdout
cnt = collections.Counter()
cur = None
infn = False
n = 0
for l in dis.splitlines():
    if ".text._ZN" in l and (".section" in l or l.startswith(".text")):
        infn = inst in l
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,5}\*/\s+[@A-Z]", l):
        n += 1
        if cur:
            cnt[cur] += 1


def find(p):
    for i, l in enumerate(src):
        if p in l:
            return i + 1
    return 10 ** 9


marks = [("helpers", 1), ("kernel-init", find("template <int KV, int CH, bool BITSET>")),
         ("expire", find("// ---- tabu expiry")), ("scan1", find("// ---- scan, phase 1")),
         ("phase2", find("// ---- phase 2: tie counts")), ("draws", find("// tenure draw (:363-365)")),
         ("locate", find("// ---- locate the sstar-th")), ("move", find("// ---- move, tenure, tabu entry")),
         ("update", find("// ---- gamma update over N(v)")), ("events", find("// events in ascending vertex order")),
         ("best", find("// ---- best (:387-390)")), ("tail", find("// ---- scratch check every 1024")),
         ("out", find("// ---------------- outputs"))]
reg = collections.Counter()
for (f, l), c in cnt.items():
    if f != "tabucol_warp.cu":
        reg["lib:" + f] += c
        continue
    r = None
    for name, ln in marks:
        if l >= ln:
            r = name
    reg[r] += c
print("instructions", n)
for k, v in reg.most_common():
    print(f"{v:6d} {k}")
