timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests6.txt 2>&1
tail -3 gpurun_out/gputests6.txt
timeout 300 bash tools/variants.sh 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench6.txt 2> gpurun_out/bench6.err
