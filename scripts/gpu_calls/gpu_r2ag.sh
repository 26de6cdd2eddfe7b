# slab ring geometry sweep: X-ring slots vs far-ring depth (rebuilds per setting)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "43 5" "41 7"; do
  set -- $cfg
  AG_NVCC_EXTRA="-DAG_SLAB_SLOTS=$1 -DAG_SLAB_FAR_SLOTS=$2" python -c "from paper_2305_17408_b200 import _build; _build.build(force=True)" > gpurun_out/build_$1_$2.log 2>&1
  echo "slots=$1 far=$2" >> gpurun_out/sweep_geom.log
  timeout 600 python scripts/slab_sweep.py --feat 256 100 48 --pairs "dense_block+coo_atomic;csr_intra_blocked+csr_inter" >> gpurun_out/sweep_geom.log 2>&1
done
echo done
