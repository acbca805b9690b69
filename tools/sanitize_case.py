"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck):
n = 64 and n = 200 RNEP, a n = 40 pencil, and an RTEST / E21 run; exits non-zero on error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1011_3077_b200 import api, inputs  # noqa: E402


def dev(x):
    return torch.as_tensor(np.asfortranarray(x)).cuda().t().contiguous().t()


h = api.Handle(256, pencil=True)
for cfg, n in ((1, 64), (5, 200)):
    p = inputs.make_config(cfg, n=n)
    _, _, _, info = h.split(dev(p.A), None, dev(p.V), max_iters=8)
    print("rnep", n, info.k, info.metric, info.status)
p = inputs.make_config(4, n=40)
_, _, _, info = h.split(dev(p.A), dev(p.B), dev(p.V), dev(p.VL), max_iters=6)
print("pencil", info.k, info.metric)
p = inputs.make_config(1)
_, _, _, info = h.split(dev(p.A), None, dev(p.V), max_iters=12, tol=1e-10, stop="e21")
print("e21", info.iters, info.metric)
_, _, _, info = h.split(dev(p.A), None, dev(p.V), max_iters=12, tol=1e-6, stop="rtest")
print("rtest", info.iters)
torch.cuda.synchronize()
print("sanitize case ok")
