cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/c4_split.py 512 > gpurun_out/c4_split.log 2>&1
echo done
