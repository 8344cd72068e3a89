set -x
ncu --set full --import-source on --clock-control none -k regex:pairwise_kernel -c 1 -o gpurun_out/r01d_distance python tools/bench_ops.py --ops distance --dist-pop 1024 > gpurun_out/ncu_d.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:greedy_init_kernel -c 1 -o gpurun_out/r01d_greedy_init python tools/bench_ops.py --ops greedy_init > gpurun_out/ncu_g.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:segsum_sorted_kernel -c 1 -o gpurun_out/r01d_segsum python tools/bench_ops.py --ops surrogate --pop-p 1024 > gpurun_out/ncu_s.log 2>&1
for r in r01d_distance r01d_greedy_init r01d_segsum; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv; ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv; done
