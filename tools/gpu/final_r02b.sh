# round-2 final evidence (after the distance restructuring): the driver's round-end
# commands (tests, smoke, both bench arms at N=1), then the bench's launch list under ncu
export PYTHONUNBUFFERED=1
bash tools/gpu/bench_full.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/bf_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu --no-e2e \
  > gpurun_out/bf_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/bf_ncu.log
