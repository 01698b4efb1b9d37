#!/bin/bash
# A/B of a dock-kernel change: paper_2303_06150_b200/libvsdock_base.so = the previous library,
# the in-tree libvsdock.so = the candidate.  Dock phase of a C4-shaped library (N ligands) at
# T = 0 (untyped) and T = 1, 2, 4 channels; the scores must be bit-identical.
set -e
mkdir -p gpurun_out
D=paper_2303_06150_b200
cp $D/libvsdock.so /tmp/libvsdock_new.so
for T in ${TS:-0 1 2 4}; do
  for v in base new; do
    if [ $v = base ]; then cp $D/libvsdock_base.so $D/libvsdock.so; else cp /tmp/libvsdock_new.so $D/libvsdock.so; fi
    TYPED=$T TAG=t${T}_$v python tools/dock_time.py ${N:-200000}
  done
  python -c "import numpy as np; a=np.load('gpurun_out/scores_t${T}_base.npy'); b=np.load('gpurun_out/scores_t${T}_new.npy'); print('T=$T bit-identical', np.array_equal(a,b))"
done
cp /tmp/libvsdock_new.so $D/libvsdock.so
