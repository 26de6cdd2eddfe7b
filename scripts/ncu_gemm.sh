# ncu --set full of the update GEMMs (C5 shapes).  Runs on the GPU box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 \
  -o gpurun_out/prof_gemm256 -f python scripts/kbench.py --feat 256 --only gemm > gpurun_out/ncu_gemm256.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 \
  -o gpurun_out/prof_gemmdh48 -f python scripts/kbench.py --feat 256 --only gemm_dh48 > gpurun_out/ncu_gemmdh48.log 2>&1
echo done
