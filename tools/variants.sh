#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()"
for n in 200000; do
  TAG=base python tools/dock_time.py $n
  TAG=nw16 VSDOCK_MAXNW=16 python tools/dock_time.py $n
  TAG=unsorted python tools/dock_time.py $n 1 1
done
