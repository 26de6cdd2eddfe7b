# ncu source-level capture of the C5 F=256 and F=48 dense_block+coo_atomic aggregation
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for F in 256 48; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slab_kernel -c 1 \
  -o gpurun_out/prof_dc$F -f python scripts/kbench.py --feat $F --only fused_pair --pair dense_block,coo_atomic \
  > gpurun_out/ncu_dc$F.log 2>&1
done
echo done
