cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_relu_bits_gpu.py tests/test_layers_gpu.py tests/test_gemm_gpu.py -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_bits.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bits.log
timeout 600 python scripts/c3_diag.py C3 > gpurun_out/c3_diag2.log 2>&1
timeout 900 python scripts/gemm_chunk_sweep.py > gpurun_out/gemm_chunk.log 2>&1
echo done
