#!/bin/bash
# timing variants for the dock phase (not bench values)
mkdir -p gpurun_out
python tools/explore.py > gpurun_out/explore3.log 2>&1; grep -E "smoke|parity|wall|==" gpurun_out/explore3.log | tail -12
for n in 10000 200000; do
  TAG=fused python tools/dock_time.py $n
  TAG=fused_unsorted python tools/dock_time.py $n 1 1
  TAG=perbucket LPB=1 python tools/dock_time.py $n
done
