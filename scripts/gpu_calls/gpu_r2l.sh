cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_kernel -c 1 \
  -o gpurun_out/prof_band256 -f python scripts/kbench.py --feat 256 --only fused_pair --pair dense_block,coo_atomic \
  > gpurun_out/ncu_band256.log 2>&1
echo done
