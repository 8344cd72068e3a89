# round-2 final evidence: C5 per-GPU share of the config at full depth (cluster vs L2 path),
# full GPU test suite, default bench, reference arm, smoke
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --workload c5 --pop 256 --depth 200000 --no-cpu --steps 1 --warmup 3 > gpurun_out/f_c5_full_cluster.json 2> gpurun_out/f_c5_full_cluster.err
timeout 900 env MCB_NO_CLUSTER=1 python bench.py --workload c5 --pop 256 --depth 200000 --no-cpu --steps 1 --warmup 3 > gpurun_out/f_c5_full_l2.json 2> gpurun_out/f_c5_full_l2.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.txt 2>&1
