TAG=r01e bash tools/profile_round.sh > gpurun_out/prof_r01e.log 2>&1
ATOMS=65,96 timeout 300 ncu --set full --clock-control none --import-source on -k regex:dock_kernel -s 2 -c 1 -o gpurun_out/dock96_r01e python tools/dock_time.py 100000 1 1 > gpurun_out/ncu27.log 2>&1
python tools/ncu_summary.py gpurun_out/dock96_r01e.ncu-rep > gpurun_out/dock96_r01e_summary.txt 2>&1
