# per-phase cycles of the warp TabuCol kernel at the C2 steady state
export PYTHONUNBUFFERED=1
for pop in 148 1184; do
timeout 300 python tools/warp_probe.py --pop $pop --depth 50000 --reps 1 --stats > gpurun_out/phase_p$pop.txt 2>&1
done
