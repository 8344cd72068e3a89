# source-level ncu capture of the 2-CTA cluster TabuCol kernel at the C5 shape (one wave)
export PYTHONUNBUFFERED=1
CMD="python tools/phase_profile.py --cluster --nodiag --n 2000 --k 150 --pop 74 --depth 1500"
$CMD > gpurun_out/ncl_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tabucol_cluster_kernel -c 1 -o gpurun_out/ncl $CMD > gpurun_out/ncl_ncu.log 2>&1
ncu -i gpurun_out/ncl.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncl_source.csv 2>/dev/null
ncu -i gpurun_out/ncl.ncu-rep --page raw --csv > gpurun_out/ncl_raw.csv 2>/dev/null
ncu -i gpurun_out/ncl.ncu-rep --page details --csv > gpurun_out/ncl_details.csv 2>/dev/null
rm -f gpurun_out/ncl.ncu-rep
