cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -m gpu -p no:cacheprovider -x -k 2sm > gpurun_out/pytest_2sm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_2sm.log
echo done
