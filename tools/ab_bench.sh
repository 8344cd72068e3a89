# A/B throughput check of two builds of the library on one GPU box:
#   cp <lib A> ab/libA.so; cp <lib B> ab/libB.so; gpurun -- 'bash tools/ab_bench.sh'
set -e
for i in 1 2 3; do
 for v in A B; do
  cp ab/lib$v.so paper_2109_05948_b200/libmemcolor_b200.so
  touch paper_2109_05948_b200/libmemcolor_b200.so
  echo "$v $(timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read())["value"])')"
 done
done
