./tools/microbench_gather 4096 512 > gpurun_out/mb2.txt 2>&1
./tools/microbench_gather 4096 1024 >> gpurun_out/mb2.txt 2>&1
ATOMS=20,64 timeout 300 ncu --set full --clock-control none --import-source on -k regex:dock_kernel -s 2 -c 1 -o gpurun_out/dock64_base python tools/dock_time.py 100000 1 1 > gpurun_out/ncu_base.log 2>&1
