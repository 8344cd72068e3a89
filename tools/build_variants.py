"""Build A/B variants of the library: each variant is compiled with extra -D
flags into ab/lib_<name>.so (load one with MCB_LIB=ab/lib_<name>.so).  Only
the files named by VARIANT_FILES (default: the warp kernel's two files) are recompiled;
the others are linked from the in-tree build (python -m
paper_2109_05948_b200._build first).
    python tools/build_variants.py name=-DFOO=1,-DBAR=0 other=..."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2109_05948_b200 import _build as B  # noqa: E402


def build(name, defs):
    out = os.path.join(ROOT, "ab")
    os.makedirs(out, exist_ok=True)
    odir = os.path.join(out, "obj_" + name)
    os.makedirs(odir, exist_ok=True)
    ccbin = ["-ccbin", "/usr/bin/g++"] if os.path.exists("/usr/bin/g++") else []
    comp = [f for f in B.NVCC_FLAGS if f != "-shared"]
    objs = []
    files = os.environ.get("VARIANT_FILES", "tabucol_warp.cu,tabucol_warp_stats.cu").split(",")
    for src in B.sources():
        base = os.path.basename(src)
        if base not in files:
            objs.append(os.path.join(B.PKG, "build", base[:-3] + ".o"))
            continue
        obj = os.path.join(odir, base[:-3] + ".o")
        cmd = [B.nvcc(), *ccbin, *B.ARCH, *comp, *defs, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        subprocess.run(cmd, check=True, capture_output=True)
        objs.append(obj)
    lib = os.path.join(out, f"lib_{name}.so")
    subprocess.run([B.nvcc(), *ccbin, *B.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib, *objs], check=True)
    return lib


specs = [a.split("=", 1) for a in sys.argv[1:]]
with ThreadPoolExecutor(max_workers=4) as ex:
    for lib in ex.map(lambda s: build(s[0], [d for d in s[1].split(",") if d]), specs):
        print(lib)
