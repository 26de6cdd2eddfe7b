cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_layers_gpu.py tests/test_parity_gpu.py tests/test_dist_gpu.py tests/test_config_parity_gpu.py tests/test_relu_bits_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_z.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_z.log
echo done
