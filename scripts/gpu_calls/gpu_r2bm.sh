cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py fwd100 > gpurun_out/gemm_trace_fwd100b.log 2>&1
AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py dw256 > gpurun_out/gemm_trace_dw256.log 2>&1
echo done
