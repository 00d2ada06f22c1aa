for spec in "ex:4:1 24 4" "cfg:3:0 29 4" "cfg:4:1 99 9"; do
  set -- $spec
  ASDSM_STREAM3D=1 timeout 60 python -c "
import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, paper_2303_01163_b200 as pb
from test_gpu_parity import _ctx
ctx,_,_=_ctx('$1',$2,$3)
st=ctx.iterate(pb.IterateOptions(tol=0.0,max_iter=3,stagnation_window=0,rng_seed=1))
print('$1', [h.res_l2 for h in st.history], sorted(k for k in ctx.kernels() if 'stream' in k))
" >> gpurun_out/s3dbg.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/ab.txt
done
