# A/B of two warp-kernel builds (in-tree vs $OLD_LIB): warp-kernel parity on the in-tree build, then one wave at depth 50k
export PYTHONUNBUFFERED=1
timeout 500 python -m pytest tests/test_tabucol_warp_gpu.py tests/test_tabucol_gpu.py tests/test_fuzz_gpu.py -x -q -p no:cacheprovider > gpurun_out/abw_t.log 2>&1; echo "rc=$?" >> gpurun_out/abw_t.log; tail -2 gpurun_out/abw_t.log
PROBE_ARGS="--pop 1184 --depth 50000 --reps 2" bash tools/ab_bench.sh ab/lib_exp.so "$OLD_LIB"
