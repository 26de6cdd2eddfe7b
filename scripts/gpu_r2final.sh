# Round-2 measurement pass (GPU box): GPU tests, every config's bench line, the
# reference arm, step profile, ncu launch list and --set full captures, sensitivity.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py --steps 10 --warmup 3 > $O/bench_C5.log 2>&1
for c in C1 C2 C3 C4; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.log 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1
timeout 600 python scripts/step_profile.py > $O/step_profile.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-graph > $O/ncu_launch_bench.log 2>&1
# --set full captures, summarised here (the reports are too large to bring back)
R=/tmp/ncu_r2
mkdir -p $R
for F in 256 48; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slab_kernel -c 1 \
  -o $R/slab$F -f python scripts/kbench.py --feat $F --only fused_pair --pair dense_block,coo_atomic > $O/ncu_slab$F.log 2>&1
done
for w in fwd256 dh48 fwd100 dw256; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 -o $R/gemm_$w -f python scripts/gemm_one.py $w > $O/ncu_gemm_$w.log 2>&1
done
python scripts/ncu_summary.py $O/ncu_summary.json slab_dense_coo_f256=$R/slab256.ncu-rep \
  slab_dense_coo_f48=$R/slab48.ncu-rep gemm_fwd_256x256_relu_maskout=$R/gemm_fwd256.ncu-rep \
  gemm_dH_48x256_mask=$R/gemm_dh48.ncu-rep gemm_fwd_100x256_relu_maskout=$R/gemm_fwd100.ncu-rep \
  gemm_dW_256x256=$R/gemm_dw256.ncu-rep > $O/ncu_summary.log 2>&1
python scripts/ncu_lines.py $R/slab256.ncu-rep slab_kernel paper_2305_17408_b200/csrc/ag_fused.cu 40 > $O/ncu_lines_slab256.txt 2>&1
python scripts/ncu_lines.py $R/gemm_dh48.ncu-rep tc_gemm paper_2305_17408_b200/csrc/ag_gemm_tc.cu 40 > $O/ncu_lines_gemm_dh48.txt 2>&1
timeout 1200 python scripts/sensitivity.py > $O/sensitivity.jsonl 2> $O/sensitivity.log
echo done
