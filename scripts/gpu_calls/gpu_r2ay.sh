cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layers_gpu.py tests/test_config_parity_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_sk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sk.log
timeout 600 python scripts/step_profile.py --config C3 > gpurun_out/step_C3.log 2>&1
timeout 600 python scripts/step_profile.py > gpurun_out/step_C5.log 2>&1
echo done
