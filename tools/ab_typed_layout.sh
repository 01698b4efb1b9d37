#!/bin/bash
# A/B of the TYPED channel layouts (Q24): QUAD windows vs scalar windows (VSDOCK_TYPED_LAYOUT),
# dock phase of a C4-shaped library (N ligands) at T = 1, 2, 4, 8 channels; scores bit-identical.
mkdir -p gpurun_out
for T in ${TS:-1 2 3 4}; do
  for L in quad scalar; do
    VSDOCK_TYPED_LAYOUT=$L TYPED=$T TAG=t${T}_$L python tools/dock_time.py ${N:-200000}
  done
  python -c "import numpy as np; a=np.load('gpurun_out/scores_t${T}_quad.npy'); b=np.load('gpurun_out/scores_t${T}_scalar.npy'); print('T=$T bit-identical', np.array_equal(a,b))"
done
