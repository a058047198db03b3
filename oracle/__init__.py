"""CPU oracle for the ℓ0–ℓ2 branch-and-bound hot path of arXiv 2602.04551.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
(paper_2602_04551_b200) never imports it and shares no code with it; the two
meet only through the seeded generators in synth/.

Plain numpy, float64, written to be checked against PAPER.md by eye.  See
oracle/l0l2_oracle.py for the per-function citations and DESIGN.md
"Readings of the paper" for every place the paper is silent or inconsistent.
"""
from .l0l2_oracle import *  # noqa: F401,F403
