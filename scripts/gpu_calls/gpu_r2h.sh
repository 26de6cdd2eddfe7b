cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/slab_sweep.py --feat 256 100 48 > gpurun_out/sweep_now.log 2>&1
timeout 600 python scripts/gemm_epi.py > gpurun_out/gemm_epi.log 2>&1
timeout 600 python scripts/step_profile.py > gpurun_out/step_profile.log 2>&1
timeout 900 python -m pytest tests/test_slab_gpu.py tests/test_relu_bits_gpu.py tests/test_dense_tc_gpu.py tests/test_dropin_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_h.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_h.log
echo done
