# round-2 re-entry: full GPU suite, C5 bench (both arms), sensitivity table, step profile
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 python scripts/step_profile.py > gpurun_out/step_profile.log 2>&1
timeout 1200 python scripts/sensitivity.py > gpurun_out/sensitivity.json 2> gpurun_out/sensitivity.log
echo done
