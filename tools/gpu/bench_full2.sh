export PYTHONUNBUFFERED=1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bf2_bench.json 2> gpurun_out/bf2_bench.err
timeout 1200 python tools/bench_generation.py --depth 100000 --gens 2 > gpurun_out/bf2_gen.txt 2>&1
