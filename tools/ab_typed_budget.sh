#!/bin/bash
# TYPED_S window budget vs warps (Q24): smaller channel windows leave room for 20 / 18 warps.
# Dock phase of a C4-shaped library (N ligands) at T = 2, 4 for several budgets (quads of 16 B).
mkdir -p gpurun_out
for B in ${BS:-8464 7400 6400 5400}; do
  for T in ${TS:-2 4}; do
    VSDOCK_TYPED_BUDGET=$B TYPED=$T TAG=b${B}_t${T} python tools/dock_time.py ${N:-200000}
  done
done
