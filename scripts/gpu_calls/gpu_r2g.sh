cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_tc_gpu.py tests/test_slab_gpu.py tests/test_relu_bits_gpu.py tests/test_dropin_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g.log
timeout 600 python scripts/step_profile.py > gpurun_out/step_profile.log 2>&1
timeout 900 python scripts/slab_sweep.py --feat 256 100 48 --knob AG_SLAB_NO_TOPO=0,1 > gpurun_out/sweep_topo.log 2>&1
echo done
