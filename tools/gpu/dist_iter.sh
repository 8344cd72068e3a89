# distance kernel iteration: parity tests, then throughput on random and related pairs
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q -k "distance or pairwise or operators or shard or smoke or engine" > gpurun_out/pd_t.log 2>&1; tail -1 gpurun_out/pd_t.log
for rel in 0 0.1 0.3; do
timeout 300 python tools/bench_ops.py --ops distance --dist-pop 4096 --dist-related $rel 2>&1 | tail -1 | cut -c1-200
done
# A/B against a previous build (MCB_LIB), when given
if [ -n "$OLD_LIB" ]; then for rel in 0 0.1 0.3; do
MCB_LIB=$OLD_LIB timeout 300 python tools/bench_ops.py --ops distance --dist-pop 4096 --dist-related $rel 2>&1 | tail -1 | cut -c1-200
done; fi
