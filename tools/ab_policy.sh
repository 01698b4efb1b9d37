#!/bin/bash
# Dock-phase A/B of the class policy on the C4-shaped mix (default policy vs 16-warp-first), and
# per class; then the bench line
mkdir -p gpurun_out
TAG=default python tools/dock_time.py ${N:-200000}
VSDOCK_POLICY="4:16,4:13,4:12,4:10,4:8" TAG=nw16 python tools/dock_time.py ${N:-200000}
python -c "import numpy as np; a=np.load('gpurun_out/scores_default.npy'); b=np.load('gpurun_out/scores_nw16.npy'); print('bit-identical', np.array_equal(a,b))"
for cls in "20,32" "33,64" "65,96" "97,128" "129,160"; do ATOMS=$cls TAG="c$cls" python tools/dock_time.py ${N:-200000} 1 1; done
