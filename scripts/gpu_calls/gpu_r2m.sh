cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/slab_sweep.py --feat 256 --pairs "dense_block+coo_atomic" --knob AG_SLAB_DEBUG=0,1,2,4,3,7 > gpurun_out/sweep_band_dbg.log 2>&1
AG_BAND=0 timeout 900 python scripts/slab_sweep.py --feat 256 --pairs "dense_block+coo_atomic" --knob AG_SLAB_DEBUG=0,1,2,4,3,7 > gpurun_out/sweep_slab_dbg.log 2>&1
echo done
