# cluster TabuCol kernel: parity tests, then C5 throughput (cluster vs the L2 CTA path)
timeout 900 python -m pytest tests/test_tabucol_cluster_gpu.py tests/test_config_shapes_gpu.py -x -q > gpurun_out/cl_tests.log 2>&1
tail -5 gpurun_out/cl_tests.log
for v in "" "MCB_NO_CLUSTER=1"; do
  echo "== $v"; env $v MCB_VERBOSE=1 timeout 600 python bench.py --workload c5 --depth 5000 --no-cpu --steps 2 --warmup 3 2>&1 | grep -E "mcb\]|\"metric\"" | tail -3 | cut -c1-600
done
