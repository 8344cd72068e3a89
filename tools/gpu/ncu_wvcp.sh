# ncu --set full of the WVCP kernel at the config-3 (C4) shape, one wave (592 individuals)
export PYTHONUNBUFFERED=1
CMD="python tools/wvcp_probe.py --pop 592 --depth 2000 --rounds 1"
$CMD > gpurun_out/wv_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:wvcp_kernel -c 1 -o gpurun_out/wv_prof $CMD > gpurun_out/wv_ncu.log 2>&1
ncu -i gpurun_out/wv_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/wv_source.csv 2>/dev/null
ncu -i gpurun_out/wv_prof.ncu-rep --page raw --csv > gpurun_out/wv_raw.csv 2>/dev/null
ncu -i gpurun_out/wv_prof.ncu-rep --page details --csv > gpurun_out/wv_details.csv 2>/dev/null
rm -f gpurun_out/wv_prof.ncu-rep
