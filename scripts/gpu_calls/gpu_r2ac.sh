cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in fwd256 dh48 fwd100 dw256; do
AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py $w > gpurun_out/gemm_trace_$w.log 2>&1
done
echo done
