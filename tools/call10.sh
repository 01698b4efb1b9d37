TAG=r01d bash tools/profile_round.sh > gpurun_out/prof_r01d.log 2>&1
python tools/ncu_summary.py gpurun_out/dock_r01d.ncu-rep > gpurun_out/dock_r01d_summary.txt 2>&1
