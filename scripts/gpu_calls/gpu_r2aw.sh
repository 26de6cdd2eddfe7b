cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --force-dist --steps 3 --warmup 3 > gpurun_out/bench_forcedist.log 2>&1; echo "rc=$?" >> gpurun_out/bench_forcedist.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --force-dist --config C3 --steps 3 --warmup 3 > gpurun_out/bench_forcedist_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_forcedist_c3.log
echo done
