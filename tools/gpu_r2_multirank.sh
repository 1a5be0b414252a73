cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TGA_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_bench_2rank_shared.json 2> gpurun_out/r2_bench_2rank_shared.err; echo rc=$?
tail -c 600 gpurun_out/r2_bench_2rank_shared.json; tail -5 gpurun_out/r2_bench_2rank_shared.err
