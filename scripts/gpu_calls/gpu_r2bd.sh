cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_band_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_band.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_band.log
echo done
