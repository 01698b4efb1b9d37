for pol in "2:16" "4:8" "2:8"; do VSDOCK_POLICY=$pol ATOMS=97,120 TAG=c128_$pol python tools/dock_time.py 200000 1 1; done > gpurun_out/pol4.txt 2>&1
ATOMS=20,64 timeout 300 ncu --set full --clock-control none --import-source on -k regex:dock_kernel -s 2 -c 1 -o gpurun_out/dock64_v2 python tools/dock_time.py 100000 1 1 > gpurun_out/ncu4a.log 2>&1
ATOMS=97,120 timeout 300 ncu --set full --clock-control none --import-source on -k regex:dock_kernel -s 2 -c 1 -o gpurun_out/dock128_v2 python tools/dock_time.py 100000 1 1 > gpurun_out/ncu4b.log 2>&1
