cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "" "AG_TC_ONEACC=1" "AG_TC_CL=1" "AG_TC_EXP=4" "AG_TC_EXP=1" "AG_TC_EXP=32" "AG_TC_EXP=16" "AG_TC_ONEACC=1 AG_TC_EXP=4"; do
  echo "== $cfg" >> gpurun_out/gemm_knobs.log
  env $cfg timeout 300 python scripts/gemm_epi.py >> gpurun_out/gemm_knobs.log 2>&1
done
AG_TC_TRACE=1 timeout 300 python -c "
import torch, sys; sys.path.insert(0,'.')
from paper_2305_17408_b200 import kernels as K
V=2449029
q=torch.randn((V,48),device='cuda'); w48=torch.randn((256,48),device='cuda'); out=torch.empty((V,256),device='cuda')
h=torch.randn((V,256),device='cuda'); w=torch.randn((256,256),device='cuda'); hb=K.relu_bits(h)
K.gemm(q, w48, out, trans_b=True, relu_mask_bits=hb); torch.cuda.synchronize()
K.gemm(h, w, out, relu=True); torch.cuda.synchronize()
" > gpurun_out/gemm_trace.log 2>&1
echo done
