# evidence for profiles/: phase breakdown + ncu --set full of the cluster kernel at C5 (one wave) + launch list of the c5 bench
export PYTHONUNBUFFERED=1
timeout 300 python tools/phase_profile.py --cluster --nodiag --n 2000 --k 150 --pop 74 --depth 5000 > gpurun_out/r02_c5_cluster_phases.txt 2>&1
timeout 300 env MCB_NO_CLUSTER=1 python tools/phase_profile.py --nodiag --n 2000 --k 150 --pop 256 --depth 3000 > gpurun_out/r02_c5_l2_phases.txt 2>&1
CMD="python tools/phase_profile.py --cluster --nodiag --n 2000 --k 150 --pop 74 --depth 1500"
ncu --set full --import-source on --clock-control none -k regex:tabucol_cluster_kernel -c 1 -o gpurun_out/ncl $CMD > gpurun_out/ncl_ncu.log 2>&1
ncu -i gpurun_out/ncl.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncl_source.csv 2>/dev/null
ncu -i gpurun_out/ncl.ncu-rep --page raw --csv > gpurun_out/ncl_raw.csv 2>/dev/null
ncu -i gpurun_out/ncl.ncu-rep --page details --csv > gpurun_out/ncl_details.csv 2>/dev/null
rm -f gpurun_out/ncl.ncu-rep
timeout 600 python bench.py --workload c5 --depth 5000 --no-cpu --steps 2 --warmup 3 > gpurun_out/r02_c5_bench.json 2>gpurun_out/r02_c5_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c5_launches.csv python bench.py --workload c5 --depth 2000 --no-cpu --steps 1 --warmup 3 > /dev/null 2>&1
