# dense + coo consumer-count sweep (rebuilds per setting)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for n in 8 10 12 14; do
  AG_NVCC_EXTRA="-DAG_SLAB_COO_CONS=$n" python -c "from paper_2305_17408_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "cons=$n" >> gpurun_out/sweep_cons.log
  timeout 600 python scripts/slab_sweep.py --feat 256 48 --pairs "dense_block+coo_atomic" >> gpurun_out/sweep_cons.log 2>&1
done
echo done
