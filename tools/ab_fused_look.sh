#!/bin/bash
# A/B of the fused multi-site ring (f1): paper_2303_06150_b200/libvsdock_base.so (previous) vs the
# in-tree library; C5-shaped campaign (N ligands x 4 pockets), per-pocket and fused launches.
mkdir -p gpurun_out
D=paper_2303_06150_b200
cp $D/libvsdock.so /tmp/libvsdock_new.so
for v in base new; do
  if [ $v = base ]; then cp $D/libvsdock_base.so $D/libvsdock.so; else cp /tmp/libvsdock_new.so $D/libvsdock.so; fi
  echo "== $v"
  VSDOCK_CLUSTER_LOG=1 python tools/fused_time.py ${N:-300000} 1 2>&1 | grep -E "fused=|size 2"
  python tools/fused_time.py ${N:-300000} 0
done
cp /tmp/libvsdock_new.so $D/libvsdock.so
