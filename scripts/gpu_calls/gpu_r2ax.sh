cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gather_gpu.py tests/test_slab_gpu.py tests/test_parity_gpu.py tests/test_layers_gpu.py tests/test_config_parity_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gp.log
for c in C1 C2 C3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gp_$c.log 2>&1; done
echo done
