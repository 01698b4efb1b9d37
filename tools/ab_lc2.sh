#!/bin/bash
# per-class dock phase vs (warps, ligands per round)
mkdir -p gpurun_out
run() { ATOMS=$1 VSDOCK_POLICY=$2 VSDOCK_LC=$3 TAG=x python tools/dock_time.py ${N:-150000} 1 1 | sed "s/^/$1 pol=$2 lc=$3 /" | cut -c1-120; }
run 20,32 4:16 1; run 20,32 4:16 2; run 20,32 4:16 4
run 33,64 4:16 1; run 33,64 4:16 2; run 33,64 4:16 3
run 97,128 4:13 1; run 97,128 4:12 2; run 97,128 4:12 1; run 97,128 4:10 2
run 129,150 4:10 1; run 129,150 4:8 2
