# Full measurement pass for the profiles: C5 bench (with the CPU baseline), C1-C4 benches,
# the ncu launch list of one C5 bench step, and the step profile.  Runs on the GPU box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
done
timeout 900 python scripts/step_profile.py > gpurun_out/step_profile.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch_bench.log 2>&1
echo done
