"""Independent check of k for the large configs: count eigenvalues strictly inside the
unit circle with LAPACK (numpy eig / scipy QZ) on the same seeded inputs.  Writes a JSON
line per config.  Test-side tool (library eigensolvers as ground truth), CPU only."""
import json
import sys
import time

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1011_3077_b200 import inputs  # noqa: E402

for cfg in [int(c) for c in sys.argv[1:]]:
    t0 = time.time()
    p = inputs.make_config(cfg)
    if p.B is None:
        lam = np.linalg.eigvals(p.A)
    else:
        lam = sla.eigvals(p.A, p.B, overwrite_a=True, overwrite_b=True, check_finite=False)
    mod = np.abs(lam)
    out = {"config": cfg, "n": p.n, "k_inside": int(np.sum(mod < 1)),
           "min_dist_to_circle": float(np.min(np.abs(mod[np.isfinite(mod)] - 1))),
           "seconds": time.time() - t0}
    print(json.dumps(out), flush=True)
