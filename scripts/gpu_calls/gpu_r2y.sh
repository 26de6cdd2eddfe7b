cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
echo "== BK32" >> gpurun_out/gemm_bk.log
timeout 300 python scripts/gemm_epi.py >> gpurun_out/gemm_bk.log 2>&1
AG_NVCC_EXTRA="-DAG_TC_BK=16" python -c "from paper_2305_17408_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
echo "== BK16" >> gpurun_out/gemm_bk.log
timeout 300 python scripts/gemm_epi.py >> gpurun_out/gemm_bk.log 2>&1
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -m gpu -p no:cacheprovider -x >> gpurun_out/gemm_bk.log 2>&1
AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py dh48 > gpurun_out/gemm_trace_dh48_bk16.log 2>&1
echo done
