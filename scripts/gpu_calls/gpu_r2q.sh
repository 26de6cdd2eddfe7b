# band kernel consumer / dense warp split sweep (rebuilds on the box per setting)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "24 4" "22 8" "26 2" "16 4"; do
  set -- $cfg
  AG_NVCC_EXTRA="-DAG_BAND_CONS=$1 -DAG_BAND_DENSE=$2" python -c "from paper_2305_17408_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "cons=$1 dense=$2" >> gpurun_out/sweep_bandcfg.log
  timeout 600 python scripts/slab_sweep.py --feat 256 48 --pairs "dense_block+coo_atomic" >> gpurun_out/sweep_bandcfg.log 2>&1
done
echo done
