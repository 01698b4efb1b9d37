#!/bin/bash
# dock phase vs ligands per round (VSDOCK_LC) on the QUAD layout
mkdir -p gpurun_out
for lc in 1 2 3 4; do VSDOCK_LC=$lc TAG=lc$lc python tools/dock_time.py ${N:-200000}; done
for lc in 1 2; do ATOMS=65,96 VSDOCK_LC=$lc TAG=c96lc$lc python tools/dock_time.py ${N:-200000} 1 1; done
python -c "import numpy as np; a=np.load('gpurun_out/scores_lc1.npy'); b=np.load('gpurun_out/scores_lc2.npy'); print('bit-identical lc1 vs lc2', np.array_equal(a,b))"
