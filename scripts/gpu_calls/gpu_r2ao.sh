cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_dropin_gpu.py tests/test_config_parity_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gather.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gather.log
timeout 900 python scripts/c4_split.py 512 > gpurun_out/c4_split2.log 2>&1
AG_COO_ATOMIC=1 timeout 900 python scripts/c4_split.py 512 > gpurun_out/c4_split2_atomic.log 2>&1
echo done
