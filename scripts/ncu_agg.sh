# ncu --set full of one fused aggregation launch (C5, F=256) for the given pair,
# normal and with the reductions skipped (AG_SLAB_DEBUG=1).  Runs on the GPU box.
#   bash scripts/ncu_agg.sh dense_block,csr_inter tag
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PAIR=${1:-dense_block,csr_inter}
TAG=${2:-agg}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slab_kernel -c 1 \
  -o gpurun_out/prof_${TAG} -f python scripts/kbench.py --feat 256 --only fused_pair --pair $PAIR \
  > gpurun_out/ncu_${TAG}.log 2>&1
AG_SLAB_DEBUG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:slab_kernel -c 1 \
  -o gpurun_out/prof_${TAG}_nr -f python scripts/kbench.py --feat 256 --only fused_pair --pair $PAIR \
  > gpurun_out/ncu_${TAG}_nr.log 2>&1
echo done
