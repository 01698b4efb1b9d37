#!/bin/bash
# One GPU call: bench (JSON), ncu launch list of a bench step, ncu --set full of one dock launch,
# and per-launch DRAM bytes of the dock kernels of one step (roofline traffic).
set -x
TAG=${TAG:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
# launch list of one full step (not a bench value: serialised, cold caches)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-unsorted --no-cpu-baseline > /dev/null 2>&1
# full capture of one dock launch (the heaviest class) of a 200k-ligand library
ncu --set full --clock-control none --import-source on -k regex:dock_kernel -s 6 -c 1 -o gpurun_out/dock_$TAG \
    python tools/dock_time.py 200000 > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
