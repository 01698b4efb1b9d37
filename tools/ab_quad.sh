#!/bin/bash
# A/B of the dock phase: QUAD (default) vs the scalar layouts (VSDOCK_GRID_MODE=scalar), C4-shaped
mkdir -p gpurun_out
for m in quad scalar; do VSDOCK_GRID_MODE=$m TAG=$m python tools/dock_time.py ${N:-200000}; done
python -c "import numpy as np; a=np.load('gpurun_out/scores_quad.npy'); b=np.load('gpurun_out/scores_scalar.npy'); print('bit-identical', np.array_equal(a,b))"
for m in quad scalar; do ATOMS=65,96 VSDOCK_GRID_MODE=$m TAG=c96$m python tools/dock_time.py ${N:-200000} 1 1; done
