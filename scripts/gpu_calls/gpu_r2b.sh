cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./build/mbar_control > gpurun_out/mbar_plain.log 2>&1; echo "rc=$?" >> gpurun_out/mbar_plain.log
timeout 300 compute-sanitizer --tool racecheck ./build/mbar_control > gpurun_out/mbar_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/mbar_racecheck.log
timeout 600 python scripts/gemm_kerr.py > gpurun_out/gemm_kerr.log 2>&1
bash scripts/ncu_agg.sh dense_block,coo_atomic dc
timeout 600 python -m pytest tests/test_config_parity_gpu.py -q -m gpu -p no:cacheprovider -k "C1 or C2" > gpurun_out/pytest_cfg.log 2>&1
echo done
