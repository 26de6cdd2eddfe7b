cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
timeout 900 python scripts/halo_report.py > gpurun_out/halo_c5.json 2> gpurun_out/halo_c5.log
echo done
