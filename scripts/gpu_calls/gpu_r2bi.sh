cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/host_overhead.py > gpurun_out/host_overhead.log 2>&1
echo done
