cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py dh48 > gpurun_out/gemm_trace_dh48.log 2>&1
AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py fwd100 > gpurun_out/gemm_trace_fwd100.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o gpurun_out/prof_dh48 -f python scripts/gemm_one.py dh48 > gpurun_out/ncu_dh48.log 2>&1
echo done
