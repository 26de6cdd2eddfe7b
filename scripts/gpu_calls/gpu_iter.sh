# usage: bash scripts/gpu_iter.sh [tests] [smoke] [bench] [kbench] [ncu] ...  (runs on the GPU box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for what in "$@"; do
case $what in
tests)
  timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log ;;
smoke)
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log ;;
bench)
  timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1 ;;
benchnocpu)
  timeout 1500 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1 ;;
ncu)
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1 ;;
ncufused)
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:slab_kernel -c 1 -o gpurun_out/prof_fused -f python scripts/kbench.py --feat 256 --only fused_pair > gpurun_out/ncu_fused.log 2>&1 ;;
kbench)
  timeout 900 python scripts/kbench.py > gpurun_out/kbench.log 2>&1 ;;
esac
done
echo done
