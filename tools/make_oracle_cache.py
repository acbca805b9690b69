"""Write tests/golden/oracle_cache/<case>.npz: the ORACLE's results for the full-code-path
twins (tests/oracle_cache.py CASES).  Calls only oracle/ and the seeded input generators --
never the CUDA path -- so every cached value is the oracle's (task rule: a stored expected
value is written by a committed script that calls only oracle/).

  python tools/make_oracle_cache.py [case ...]      (default: every case)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import oracle_cache  # noqa: E402


def main(names):
    for name in names or list(oracle_cache.CASES):
        t0 = time.time()
        path = oracle_cache.make(name)
        print(f"{name}: {time.time() - t0:.1f} s -> {os.path.relpath(path, ROOT)}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
