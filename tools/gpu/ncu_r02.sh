# round-2 evidence: the bench's launch list, a fresh WVCP capture
export PYTHONUNBUFFERED=1
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r02_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r02_ncu_launch.log 2>&1
bash tools/gpu/ncu_wvcp.sh
