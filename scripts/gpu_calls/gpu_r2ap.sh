cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/c5_nonfused.py > gpurun_out/c5_nonfused.log 2>&1
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.log 2>&1
echo done
