timeout 600 python -m pytest tests -m gpu -x -q -k "distance or pairwise or operators or shard" > gpurun_out/pd_t.log 2>&1; tail -1 gpurun_out/pd_t.log
timeout 300 python tools/bench_ops.py --ops distance --dist-pop 4096 2>&1 | tail -1 | cut -c1-120
