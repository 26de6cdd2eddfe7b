cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/gemm_kerr.py > gpurun_out/gemm_kerr2.log 2>&1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_config_parity_gpu.py tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c.log
echo done
