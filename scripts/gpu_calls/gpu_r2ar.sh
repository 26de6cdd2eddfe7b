cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -x -k "coo_gather" > gpurun_out/pytest_cg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cg.log
echo done
