cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R=/tmp/ncu_c4
mkdir -p $R
timeout 900 ncu --set full --clock-control none -k regex:"tc_gemm|coo_gather" -c 4 -o $R/c4 -f python scripts/c4_kernels_once.py > gpurun_out/ncu_c4.log 2>&1
ncu -i $R/c4.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct > gpurun_out/ncu_c4_raw.csv 2>&1
echo done
