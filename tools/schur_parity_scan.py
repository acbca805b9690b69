"""GPU vs oracle decisions of sdc_schur on candidate parity cases (run on a B200): block lists and
(splits, failed attempts, unsplit) for cases whose oracle decisions survive 2e-14 relative input
noise (tests/test_oracle_schur.py) and for two that only survive 4e-16 (reading Q20b).
Output of round 2: profiles/r02_experiments/schur_batched_parity_scan.txt."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle
from paper_1011_3077_b200 import api, inputs
cases = [(96,1,6),(96,1,25),(96,1,34),(128,1,13),(128,1,19),(128,1,26),(160,2,32),(128,1,1),(200,2,7)]
h = api.Handle(256)
for n, leaf, seed in cases:
    A,_,_ = inputs.normal_random_eigs(n, 15+n, 16+n)
    Ad = torch.as_tensor(np.asfortranarray(A)).cuda().t().contiguous().t()
    Q,T,blocks,info = h.schur(Ad, leaf=leaf, seed=seed)
    o = oracle.schur(A, leaf=leaf, seed=seed)
    print(n, leaf, seed, "blocks_equal", blocks == o.blocks, "gpu", (info["splits"], info["failed_attempts"], info["unsplit"]),
          "orc", (o.splits, o.failed_attempts, o.unsplit), flush=True)
