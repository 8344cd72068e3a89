# C3 shape: warp kernel (default) vs the 2-CTA cluster kernel (forced), 16384 individuals x 2000 iterations
for a in "" "--cluster" ; do for nt in 256 512; do
 echo "== $a nt=$nt"; MCB_CL_NT=$nt MCB_VERBOSE=1 timeout 600 python tools/phase_profile.py $a --nodiag --n 1000 --k 83 --pop 16384 --depth 2000 2>&1 | grep -E "iterations|mcb\]" | head -3
 [ -z "$a" ] && break
done; done
