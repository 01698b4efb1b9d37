VSDOCK_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --ligands 200000 --no-unsorted > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
tail -3 gpurun_out/bench_2rank.err
timeout 900 python bench.py --steps 3 --warmup 3 --ligands 200000 --no-unsorted --no-cpu-baseline > gpurun_out/bench_1rank_200k.json 2> gpurun_out/bench_1rank_200k.err
