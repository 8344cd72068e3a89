export PYTHONUNBUFFERED=1
timeout 900 python tools/warp_probe.py --n 1000 --k 83 --pop 296 --depth 20000 --warm 20000 --reps 1 --var 'warp:MCB_GROUP_NW=0' --var 'g2:MCB_GROUP_NW=2' --var 'g4:MCB_GROUP_NW=4' --var 'g1:MCB_GROUP_NW=1' > gpurun_out/c3g.txt 2>&1
timeout 900 python tools/warp_probe.py --n 500 --k 48 --pop 1184 --depth 20000 --warm 20000 --reps 1 --var 'warp:MCB_GROUP_NW=0' --var 'g2:MCB_GROUP_NW=2' > gpurun_out/c2g.txt 2>&1
