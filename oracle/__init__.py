"""CPU fp64 oracle for the inverse-free split step (arXiv 1011.3077).

TEST INFRASTRUCTURE ONLY.  Importable only from tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  Shares no code with the CUDA path
(paper_1011_3077_b200/); see oracle/sdc_oracle.c for the algorithm and its citations.
"""
from .oracle import *  # noqa: F401,F403
