"""Reproduce the paper's numerical experiments E1-E4 (Figures
numexp_rand and numexp_hard) on the GPU: normal / non-normal matrices split on the
imaginary axis (half plane Re z < 0 via the Moebius pencil), full split
after every IRS pass (the E21 monitor protocol of PAPER.md:597, tol = 0 so all passes run),
recording the backward error per pass.  The paper plots ||E21||_2/||A||_2; we record the
1-norm metric the algorithm selects with (Alg. 5) and, at the last pass, both norms.
Writes one JSON line per experiment to stdout."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1011_3077_b200 import api, inputs  # noqa: E402


def dev(x):
    return torch.as_tensor(np.asfortranarray(x)).cuda().t().contiguous().t()


h = api.Handle(1024)
for name, e in inputs.EXPERIMENTS.items():
    A, V, eig = e["fn"](e["n"], e["seed"], e["vseed"])
    Q, _, Ah, info = h.split(dev(A), None, dev(V), max_iters=e["passes"], tol=0.0, stop="e21",
                             region="halfplane", param=0.0, want_ahat=True)
    hist = info.hist[:, 1]
    ah = Ah.cpu().numpy()
    r = info.r
    e21_2 = float(np.linalg.norm(ah[r:, :r], 2) / np.linalg.norm(A, 2))
    first = next((j + 1 for j, m in enumerate(hist) if m <= 1e-12), None)
    print(json.dumps({
        "experiment": name, "n": e["n"], "passes": e["passes"],
        "min_dist_to_axis": float(np.min(np.abs(eig.real))),
        "k_left_true": int(np.sum(eig.real < 0)), "k": info.k, "status": info.status,
        "first_pass_metric_le_1e-12": first, "final_metric_1norm": float(hist[-1]),
        "final_E21_2norm_rel": e21_2,
        "metric_history": [float(x) for x in hist]}), flush=True)
