#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()"
n=200000
TAG=default python tools/dock_time.py $n
TAG=p2 VSDOCK_POLICY="2:32,2:16,2:8" python tools/dock_time.py $n
TAG=unsorted_default python tools/dock_time.py $n 1 1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
