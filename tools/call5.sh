timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gputests5.txt 2>&1
tail -3 gpurun_out/gputests5.txt
timeout 300 bash tools/variants.sh 2>&1 | tail -4
for pol in "4:8" "2:16"; do VSDOCK_POLICY=$pol ATOMS=97,120 TAG=c128_$pol timeout 120 python tools/dock_time.py 200000 1 1; done
timeout 600 python bench.py > gpurun_out/bench5.txt 2> gpurun_out/bench5.err
