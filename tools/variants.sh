#!/bin/bash
python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
TAG=default python tools/dock_time.py 200000
ATOMS=20,64 TAG=c64 python tools/dock_time.py 200000 1 1
ATOMS=65,96 TAG=c96 python tools/dock_time.py 200000 1 1
ATOMS=97,120 TAG=c128 python tools/dock_time.py 200000 1 1
