# cluster kernel: parity, then phases at C5 (one wave), then the c5 bench line
timeout 900 python -m pytest tests/test_tabucol_cluster_gpu.py tests/test_config_shapes_gpu.py -x -q -k "cluster or c5" > gpurun_out/cl_tests.log 2>&1
tail -3 gpurun_out/cl_tests.log
timeout 300 python tools/phase_profile.py --cluster --nodiag --n 2000 --k 150 --pop 74 --depth 5000 2>&1 | head -11
timeout 600 python bench.py --workload c5 --depth 5000 --no-cpu --steps 2 --warmup 3 2>&1 | grep '"metric"' | cut -c1-300
