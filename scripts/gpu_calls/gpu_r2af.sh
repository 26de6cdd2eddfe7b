cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "" "AG_TC_BN=128 AG_TC_ONEACC=1" "AG_TC_BN=128" "AG_TC_CL=1"; do
  echo "== $cfg" >> gpurun_out/gemm_knobs3.log
  env $cfg timeout 300 python scripts/gemm_epi.py >> gpurun_out/gemm_knobs3.log 2>&1
done
echo done
