# source-level ncu capture of the warp TabuCol kernel at the C2 steady state
export PYTHONUNBUFFERED=1
CMD="python tools/warp_probe.py --pop 1184 --depth 50000 --reps 1"
$CMD > gpurun_out/nw_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tabucol_warp_kernel -s 1 -c 1 -o gpurun_out/nw_warp $CMD > gpurun_out/nw_ncu.log 2>&1
ncu -i gpurun_out/nw_warp.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/nw_source.csv 2>/dev/null
ncu -i gpurun_out/nw_warp.ncu-rep --page raw --csv > gpurun_out/nw_raw.csv 2>/dev/null
ncu -i gpurun_out/nw_warp.ncu-rep --page details --csv > gpurun_out/nw_details.csv 2>/dev/null
rm -f gpurun_out/nw_warp.ncu-rep
