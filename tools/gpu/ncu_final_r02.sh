# final ncu --set full captures of the WVCP kernel (C4 shape, one wave) and the cluster TabuCol kernel (C5, one wave)
export PYTHONUNBUFFERED=1
bash tools/gpu/ncu_wvcp.sh
bash tools/gpu/ncu_cluster.sh
