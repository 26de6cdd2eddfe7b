cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "" "AG_TC_RAWHI=0" "" "AG_TC_RAWHI=0"; do
echo "== $cfg" >> gpurun_out/gemm_rawhi.log
env $cfg timeout 300 python scripts/gemm_epi.py >> gpurun_out/gemm_rawhi.log 2>&1
done
echo done
