"""One sdc_schur decomposition with SDC_SCHUR_TRACE=1 (one line per attempt, the oracle's
ORC_SCHUR_TRACE format): SDC_SCHUR_TRACE=1 [SDC_SCHUR_BATCH=0] python tools/schur_trace.py > gpu.txt 2> gpu.err;
diff the (o, m, att) -> (iters, status, r) maps against the oracle's trace to find the first
diverging decision."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1011_3077_b200 import api, inputs
n, leaf, seed = 128, 1, 1
A,_,_ = inputs.normal_random_eigs(n, 15+n, 16+n)
h = api.Handle(128)
Ad = torch.as_tensor(np.asfortranarray(A)).cuda().t().contiguous().t()
Q,T,blocks,info = h.schur(Ad, leaf=leaf, seed=seed)
torch.cuda.synchronize()
print(info, file=sys.stderr)
