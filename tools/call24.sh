ATOMS=20,64 timeout 300 ncu --set full --clock-control none --import-source on -k regex:dock_kernel -s 2 -c 1 -o gpurun_out/dock64_k8 python tools/dock_time.py 100000 1 1 > gpurun_out/ncu24.log 2>&1
python tools/ncu_summary.py gpurun_out/dock64_k8.ncu-rep > gpurun_out/dock64_k8_summary.txt 2>&1
