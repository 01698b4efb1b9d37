timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --config C3 --no-unsorted > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 1200 python bench.py --config C5 --no-unsorted --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
