cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/slab_sweep.py --feat 256 --pairs "dense_block+coo_atomic" --knob AG_SLAB_SLEEP=1,0 --knob AG_SLAB_CSLEEP=0,100,500 > gpurun_out/sweep_band_sleep.log 2>&1
AG_SLAB_DEBUG=7 timeout 600 python scripts/slab_sweep.py --feat 256 --pairs "dense_block+coo_atomic" --knob AG_SLAB_SLEEP=1,0 >> gpurun_out/sweep_band_sleep.log 2>&1
echo done
