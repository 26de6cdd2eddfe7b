cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/gemm_2sm_check.py > gpurun_out/gemm_2sm.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_2sm.log
AG_TC_2SM=1 timeout 300 python scripts/gemm_epi.py > gpurun_out/gemm_epi_2sm.log 2>&1
timeout 300 python scripts/gemm_epi.py > gpurun_out/gemm_epi_1sm.log 2>&1
echo done
