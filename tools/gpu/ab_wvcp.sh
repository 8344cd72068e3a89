# WVCP A/B: throughput of library builds at the C4 shape, one wave and the full population
for i in 1 2; do for lib in "$@"; do
 echo "$lib p592 $(MCB_LIB=$lib timeout 300 python tools/wvcp_probe.py --plain --pop 592 --depth 5000 --rounds 2 2>&1 | tail -1)"
 echo "$lib p8192 $(MCB_LIB=$lib timeout 300 python tools/wvcp_probe.py --plain --pop 8192 --depth 2000 --rounds 2 2>&1 | tail -1)"
done; done
