# concurrency experiment (temporary TW_MAX_WARPS = 9): the warp kernel, warps per SM 8 vs 9, at a
# latency-bound shape near the colouring threshold (n = 400, k = 48 and k = 44)
for k in 48 44; do for w in 8 9; do
  echo "== k=$k warps/SM $w"; MCB_WARPS=$w MCB_VERBOSE=1 timeout 300 python tools/warp_probe.py --n 400 --k $k --pop 9472 --depth 30000 2>&1 | grep -E "moves" | tail -1 | cut -c1-160
done; done
