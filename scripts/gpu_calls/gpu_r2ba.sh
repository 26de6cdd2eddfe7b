cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python scripts/sensitivity.py > gpurun_out/sens4.json 2> gpurun_out/sens4.log
timeout 900 python -m pytest tests/test_gather_gpu.py tests/test_slab_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_g4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g4.log
echo done
