export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t8_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/t8_pytest.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/t8_bench.json 2> gpurun_out/t8_bench.err
echo "bench rc=$?" >> gpurun_out/t8_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/t8_ref.json 2> gpurun_out/t8_ref.err
