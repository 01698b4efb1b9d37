#!/bin/bash
# One GPU call of round evidence (TAG=r02d): bench lines (C4 default, C5 with the fused multi-site
# leg, C3, C2, the typed variant, the reference arm), the ncu launch list of one bench step
# (per-kernel time + DRAM bytes), ncu --set full of the heaviest dock launch (class 96, 200k-ligand
# C4-shaped library) and of the a1 ingest kernel, summarised on the box (the reports stay in /tmp).
set -x
TAG=${TAG:-r02c}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
python bench.py --config C5 --no-e2e --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_${TAG}_c5.json 2>&1
python bench.py --config C3 --no-e2e --no-unsorted --no-cpu-baseline > gpurun_out/bench_${TAG}_c3.json 2>&1
python bench.py --config C2 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_c2.json 2>&1
python bench.py --typed 4 --no-cpu-baseline --no-unsorted > gpurun_out/bench_${TAG}_typed4.json 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2>&1
# launch list of one full step (not a bench value: serialised, cold caches)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-unsorted --no-cpu-baseline > /dev/null 2>&1
# full capture of one dock launch (class 96) of a 200k-ligand library, and of the ingest kernel
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:dock_kernel<.int.96," -s 1 -c 1 \
    -o /tmp/dock96_$TAG python tools/dock_time.py 200000 > gpurun_out/ncu_dock_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/dock96_$TAG.ncu-rep > gpurun_out/dock96_${TAG}_ncu_summary.txt 2>&1
python tools/ncu_lines.py /tmp/dock96_$TAG.ncu-rep 60 > gpurun_out/dock96_${TAG}_ncu_lines.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:ingest -s 1 -c 1 -o /tmp/ingest_$TAG \
    python tools/dock_time.py 200000 > gpurun_out/ncu_ingest_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/ingest_$TAG.ncu-rep > gpurun_out/ingest_${TAG}_ncu_summary.txt 2>&1
tail -3 gpurun_out/ncu_dock_$TAG.log
# full capture of one TYPED_S dock launch (class 96, 4 atom types)
TYPED=4 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:dock_kernel<.int.96," -s 1 -c 1 \
    -o /tmp/dock96t4_$TAG python tools/dock_time.py 200000 > gpurun_out/ncu_dock_t4_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/dock96t4_$TAG.ncu-rep > gpurun_out/dock96_typed4_${TAG}_ncu_summary.txt 2>&1
