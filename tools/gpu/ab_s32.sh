# A/B: 32-bit conflict scalars in the warp kernel; parity of the in-tree build first
export PYTHONUNBUFFERED=1
timeout 400 python -m pytest tests/test_tabucol_warp_gpu.py tests/test_tabucol_gpu.py tests/test_fuzz_gpu.py -x -q -p no:cacheprovider > gpurun_out/s32_t.log 2>&1; echo "rc=$?" >> gpurun_out/s32_t.log; tail -2 gpurun_out/s32_t.log
PROBE_ARGS="--pop 1184 --depth 50000 --reps 2" bash tools/ab_bench.sh ab/lib_s32.so ab/lib_base.so
