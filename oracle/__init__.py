"""TEST INFRASTRUCTURE ONLY — the fp64 CPU oracle for arxiv 2006.16147.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product library
(paper_2006_16147_b200/) never imports, links or executes it, and the two share
no code.  See oracle.c for the step-by-step citations of the paper.
"""
from .oracle import *  # noqa: F401,F403
