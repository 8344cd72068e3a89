# headline config: the per-GPU share of D=8192 at N = 2, 4, 8 (one B200), 50k iterations
for p in 4096 2048 1024; do
  timeout 600 python bench.py --pop $p --no-extra --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print($p, d['value'], d['ms_per_step'], d['roofline']['kernel'][:60])"
done
