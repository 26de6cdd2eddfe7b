cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_relu_bits_gpu.py tests/test_layers_gpu.py tests/test_slab_gpu.py -k "gemm or relu or layer" -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 300 python scripts/gemm_epi.py > gpurun_out/gemm_epi5.log 2>&1
AG_TC_NO_CTMA=1 timeout 300 python scripts/gemm_epi.py > gpurun_out/gemm_epi5b.log 2>&1
AG_TC_TRACE=1 timeout 300 python scripts/gemm_one.py dh48 > gpurun_out/gemm_trace_dh48.log 2>&1
echo done
