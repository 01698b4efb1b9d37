set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests3.txt 2>&1
tail -3 gpurun_out/gputests3.txt
bash tools/variants.sh > gpurun_out/var3.txt 2>&1
cat gpurun_out/var3.txt
timeout 600 python bench.py > gpurun_out/bench3.txt 2> gpurun_out/bench3.err
