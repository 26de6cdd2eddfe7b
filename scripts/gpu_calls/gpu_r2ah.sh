cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for B in 16 512; do
timeout 900 python bench.py --config C4 --comm-size $B --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4_B$B.log 2>&1
done
echo done
