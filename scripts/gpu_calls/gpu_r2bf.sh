cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/slab_sweep.py --feat 256 100 48 --pairs "dense_block+coo_atomic" --knob AG_GATHER=0,2 > gpurun_out/sweep_gather2.log 2>&1
timeout 900 python -m pytest tests/test_gather_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_g6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g6.log
echo done
