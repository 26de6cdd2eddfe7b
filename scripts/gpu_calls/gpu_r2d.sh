cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/gemm_kerr.py > gpurun_out/gemm_kerr3.log 2>&1
timeout 600 python scripts/c3_diag.py C3 > gpurun_out/c3_diag.log 2>&1
timeout 900 python scripts/slab_sweep.py --feat 256 --pairs "dense_block+coo_atomic;csr_intra_blocked+csr_inter" --knob AG_SLAB_CSLEEP=0,50,200,1000 > gpurun_out/sweep_csleep.log 2>&1
echo done
