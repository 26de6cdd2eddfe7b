cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_slab_gpu.py -q -m gpu -p no:cacheprovider -x -k "dense or coo" > gpurun_out/pytest_coo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coo.log
timeout 600 python scripts/slab_sweep.py --feat 256 100 48 --pairs "dense_block+coo_atomic" > gpurun_out/sweep_coo.log 2>&1
echo done
