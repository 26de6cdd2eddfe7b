cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_band_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_band.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_band.log
timeout 900 python scripts/slab_sweep.py --feat 256 100 48 --pairs "dense_block+coo_atomic" --knob AG_SLAB_DEBUG=0,1,7 > gpurun_out/sweep_band.log 2>&1
echo done
