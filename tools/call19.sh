timeout 600 python bench.py --no-unsorted --no-cpu-baseline --steps 3 > gpurun_out/bench19.json 2> gpurun_out/bench19.err
timeout 900 python tools/experiments.py heatmap 1000000 > gpurun_out/exp_h1m.log 2>&1
timeout 300 python tools/experiments.py heatmap 10000 > gpurun_out/exp_h10k.log 2>&1
timeout 600 python tools/experiments.py sweep 100000 > gpurun_out/exp_sweep.log 2>&1
