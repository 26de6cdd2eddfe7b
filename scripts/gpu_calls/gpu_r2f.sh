cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 600 python scripts/gemm_chunk_sweep.py > gpurun_out/gemm_chunk2.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref.log 2>&1
timeout 1800 python scripts/cpu_fullscale.py > gpurun_out/cpu_fullscale_c5.json 2> gpurun_out/cpu_fullscale.log
echo done
