# distance kernel: throughput (random and LS-like colourings) + source-level ncu
export PYTHONUNBUFFERED=1
timeout 300 python tools/bench_ops.py --ops distance --dist-pop 4096 > gpurun_out/pd_bench.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:pairwise_kernel -c 1 -o gpurun_out/npd python tools/bench_ops.py --ops distance --dist-pop 1024 > gpurun_out/npd_ncu.log 2>&1
ncu -i gpurun_out/npd.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/npd_source.csv 2>/dev/null
ncu -i gpurun_out/npd.ncu-rep --page raw --csv > gpurun_out/npd_raw.csv 2>/dev/null
rm -f gpurun_out/npd.ncu-rep
