cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist exit $?"
tail -5 gpurun_out/pytest_dist.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_trun.json 2> gpurun_out/bench_trun.err; echo "torchrun exit $?"
tail -c 600 gpurun_out/bench_trun.json; tail -3 gpurun_out/bench_trun.err
