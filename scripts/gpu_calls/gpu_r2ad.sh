cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o gpurun_out/prof_dh48b -f python scripts/gemm_one.py dh48 > gpurun_out/ncu_dh48b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o gpurun_out/prof_fwd256 -f python scripts/gemm_one.py fwd256 > gpurun_out/ncu_fwd256.log 2>&1
echo done
