"""fp64 CPU oracle for the motion-blur hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  It shares no code with paper_2602_07860_b200 (the CUDA
path); see oracle.c for what is computed and the passages each step follows.
Parity pins: tests/test_oracle_pins.py.  Parity unpinned: none of the oracle's
functions (the paper's figures are absent, so nothing is pinned to a printed image;
every function is pinned by closed forms, library routines, brute force or FD).
"""
from .oracle import *  # noqa: F401,F403
