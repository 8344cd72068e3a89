for d in 0 1; do echo "== dbg $d"; MCB_CL_DEBUG=$d timeout 300 python tools/phase_profile.py --cluster --nodiag --n 2000 --k 150 --pop 74 --depth 5000 2>&1 | grep -E "iterations|pass1|p1 work"; done
