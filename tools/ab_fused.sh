#!/bin/bash
# Fused multi-site (f1) on C5-shaped pockets: per-pocket launches vs fused clusters of size 2 and 4
mkdir -p gpurun_out
VSDOCK_CLUSTER_LOG=1 python tools/fused_time.py ${N:-300000} 0 2>&1 | tail -12
for g in 2 4; do VSDOCK_CLUSTER=$g python tools/fused_time.py ${N:-300000} 1; done
