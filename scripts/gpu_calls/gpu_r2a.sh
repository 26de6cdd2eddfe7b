# round-2 check: new parity tests + sanitizer passes on the slab kernel (GPU box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_layers_gpu.py tests/test_config_parity_gpu.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 300 python scripts/sanitize_slab.py > gpurun_out/plain_slab.log 2>&1; echo "rc=$?" >> gpurun_out/plain_slab.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_slab.py > gpurun_out/sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
echo done
