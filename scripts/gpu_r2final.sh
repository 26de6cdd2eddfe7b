# Round-2 measurement pass (GPU box): GPU tests, every config's bench line, the
# reference arm, step profile, ncu launch list and --set full captures, sensitivity.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/bench_C5.log 2>&1
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1
timeout 600 python scripts/step_profile.py > $O/step_profile.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph > $O/ncu_launch_bench.log 2>&1
for F in 256 48; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slab_kernel -c 1 \
  -o $O/prof_slab$F -f python scripts/kbench.py --feat $F --only fused_pair --pair dense_block,coo_atomic > $O/ncu_slab$F.log 2>&1
done
for w in fwd256 dh48 fwd100 dw256; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o $O/prof_gemm_$w -f python scripts/gemm_one.py $w > $O/ncu_gemm_$w.log 2>&1
done
timeout 1200 python scripts/sensitivity.py > $O/sensitivity.jsonl 2> $O/sensitivity.log
echo done
