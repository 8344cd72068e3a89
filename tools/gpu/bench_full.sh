# the driver's round-end commands: tests, smoke, both bench arms (N=1)
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/bf_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/bf_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bf_smoke.txt 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bf_ref.json 2> gpurun_out/bf_ref.err
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw --format=csv -lms 500 > gpurun_out/bf_clocks.csv &
SMI=$!
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bf_bench.json 2> gpurun_out/bf_bench.err
kill $SMI
