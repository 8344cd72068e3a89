# distance kernel debug: one test file under a short timeout, then throughput
export PYTHONUNBUFFERED=1
timeout 120 python -m pytest tests/test_operators_gpu.py -x -q -p no:cacheprovider > gpurun_out/pdd_ops.log 2>&1; echo "ops rc=$?" >> gpurun_out/pdd_ops.log
for rel in 0 0.1 0.3; do
timeout 60 python tools/bench_ops.py --ops distance --dist-pop 4096 --dist-related $rel 2>&1 | tail -1 | cut -c1-100
done
