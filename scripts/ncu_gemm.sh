# ncu --set full of the update GEMMs (C5 shapes).  Runs on the GPU box.
#   bash scripts/ncu_gemm.sh [only=gemm|gemm_dh48] [tag] [extra env assignments...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ONLY=${1:-gemm}
TAG=${2:-$ONLY}
shift 2
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -c 1 \
  -o gpurun_out/prof_$TAG -f python scripts/kbench.py --feat 256 --only $ONLY > gpurun_out/ncu_$TAG.log 2>&1
echo done
