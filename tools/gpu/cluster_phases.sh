# cluster kernel phase breakdown at the C5 shape (one wave: 74 clusters), early and deeper
for d in 2000 5000; do
  echo "== depth $d"; timeout 300 python tools/phase_profile.py --cluster --nodiag --n 2000 --k 150 --pop 74 --depth $d 2>&1 | tail -10
done
for nt in 256 1024; do echo "== nt $nt"; MCB_CL_NT=$nt timeout 300 python tools/phase_profile.py --cluster --nodiag --n 2000 --k 150 --pop 74 --depth 5000 2>&1 | tail -10; done
