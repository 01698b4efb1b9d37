timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests8.txt 2>&1
tail -3 gpurun_out/gputests8.txt
timeout 300 bash tools/variants.sh 2>&1 | tail -4
