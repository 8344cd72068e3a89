export PYTHONUNBUFFERED=1
CMD="python tools/warp_probe.py --pop 1184 --depth 10000 --reps 1"
MCB_GROUP_NW=1 $CMD > gpurun_out/t7_plain.log 2>&1 && \
MCB_GROUP_NW=1 ncu --set full --import-source on --clock-control none -k regex:tabucol_group_kernel -s 1 -c 1 -o gpurun_out/t7_g1 $CMD > gpurun_out/t7_ncu.log 2>&1
ncu -i gpurun_out/t7_g1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/t7_source.csv 2>/dev/null
ncu -i gpurun_out/t7_g1.ncu-rep --page raw --csv > gpurun_out/t7_raw.csv 2>/dev/null
rm -f gpurun_out/t7_g1.ncu-rep
