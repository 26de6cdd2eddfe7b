cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/slab_sweep.py --feat 256 100 48 --pairs "dense_block+coo_atomic" --knob AG_GATHER=0,2 > gpurun_out/sweep_gather.log 2>&1
echo done
