#!/bin/bash
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TAG=default python tools/dock_time.py 200000
ATOMS=20,64 TAG=c64 python tools/dock_time.py 200000 1 1
ATOMS=65,96 TAG=c96 python tools/dock_time.py 200000 1 1
ATOMS=97,120 TAG=c128 python tools/dock_time.py 200000 1 1
ATOMS=65,96 TAG=c96p2 VSDOCK_POLICY=2:16 python tools/dock_time.py 200000 1 1
