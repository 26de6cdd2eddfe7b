# Time the fused aggregation with parts of the pipeline switched off (AG_SLAB_DEBUG bits;
# values are garbage then).  Runs on the GPU box.
cd $GRAFT_REPO_ROOT
for dbg in ${DBGS:-0 1 3 5 7 9 15 2 4}; do
AG_SLAB_DEBUG=$dbg timeout 600 python scripts/kbench.py --suite agg --feat 256 > gpurun_out/kb_dbg$dbg.log 2>&1
python - $dbg <<EOP
import json,sys
t=open("gpurun_out/kb_dbg%s.log"%sys.argv[1]).read()
d=json.loads(t[t.index("{"):])
m=d["F256"]["ms"]
print("dbg", sys.argv[1], {k:m[k] for k in ("csr_intra_blocked+csr_inter","dense_block+csr_inter","dense_block+coo_atomic")})
EOP
done
