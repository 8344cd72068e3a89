# A/B of two distance-kernel builds (in-tree vs $OLD_LIB): parity tests on the in-tree build, then throughput
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_operators_gpu.py tests/test_limits_gpu.py -x -q -p no:cacheprovider > gpurun_out/abd_t.log 2>&1; echo "rc=$?" >> gpurun_out/abd_t.log; tail -2 gpurun_out/abd_t.log
for rel in 0 0.1; do for lib in "" "$OLD_LIB"; do
MCB_LIB=$lib timeout 60 python tools/bench_ops.py --ops distance --dist-pop 4096 --dist-related $rel 2>&1 | tail -1 | cut -c1-60
done; done
