cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "" "AG_TC_CL=1" "AG_TC_CL=2" "AG_TC_ONEACC=1" "AG_TC_BN=32" "AG_TC_BN=128"; do
  echo "== $cfg" >> gpurun_out/gemm_small.log
  env $cfg timeout 300 python scripts/gemm_small.py >> gpurun_out/gemm_small.log 2>&1
done
echo done
