# CTA kernel (L2 path and fallbacks): parity, then C5 L2-path phases and full-depth bench
timeout 900 python -m pytest tests -m gpu -x -q -k "tabucol or config_shapes or limits or fuzz or async or production or engine" > gpurun_out/cta_t.log 2>&1; tail -2 gpurun_out/cta_t.log
MCB_NO_CLUSTER=1 timeout 600 python tools/phase_profile.py --nodiag --n 2000 --k 150 --pop 256 --depth 50000 2>&1 | head -11
timeout 900 env MCB_NO_CLUSTER=1 python bench.py --workload c5 --pop 256 --depth 200000 --no-cpu --steps 1 --warmup 3 2>/dev/null | cut -c1-200
