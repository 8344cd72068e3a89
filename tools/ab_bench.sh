# A/B throughput of library builds on one GPU box, each loaded through
# MCB_LIB (the in-tree library is never touched):
#   python tools/build_variants.py a=-DX=0 b=-DX=1
#   gpurun -- 'bash tools/ab_bench.sh ab/lib_a.so ab/lib_b.so'
# extra warp_probe arguments via PROBE_ARGS (default: one wave at depth 50k)
ARGS=${PROBE_ARGS:---pop 1184 --depth 50000 --reps 3}
for i in 1 2; do
 for lib in "$@"; do
  echo "$lib $(MCB_LIB=$lib timeout 300 python tools/warp_probe.py $ARGS 2>/dev/null | tail -1)"
 done
done
