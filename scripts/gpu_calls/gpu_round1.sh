cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 --cpu-rows 20000 > gpurun_out/bench_c5.log 2>&1
echo done
