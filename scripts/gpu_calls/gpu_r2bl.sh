# C1-C4 bench lines with the host baseline (full epochs for C1-C3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
for c in C1 C2 C3 C4; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/final2/bench_$c.log 2>&1
done
echo done
