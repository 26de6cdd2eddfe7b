cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py fwd256 > gpurun_out/gemm_trace_fwd256.log 2>&1
AG_TC_2SM=1 AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py fwd256 > gpurun_out/gemm_trace_fwd256_2sm.log 2>&1
echo done
