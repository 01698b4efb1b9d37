#!/bin/bash
# A/B of warps per CTA for the 32 / 64 atom classes (QUAD, K = 8): 16 / 20 / 24 warps, LC = 1 or 2
mkdir -p gpurun_out
for cls in "20,32" "33,64"; do
  for pol in "4:16" "4:20" "4:24"; do
    for lc in 1 2; do
      ATOMS=$cls VSDOCK_POLICY=$pol VSDOCK_LC=$lc TAG="a$cls-p$pol-lc$lc" python tools/dock_time.py ${N:-200000} 1 1
    done
  done
done
for T in 1 2 4; do TYPED=$T TAG=typed$T python tools/dock_time.py ${N:-200000}; done
