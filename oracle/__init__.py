"""TEST INFRASTRUCTURE ONLY — the serial fp64 CPU oracle of the ZPIC em2d step.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It shares no code with paper_2106_12485_b200/ (the CUDA path), and the
product path never imports it.  See oracle/zpic_oracle.c for the per-stage citations and
oracle/sim.py for the step order.

Parity pins: every function here is pinned by -m "not gpu" tests in tests/test_oracle_*.py
against closed forms, library routines and brute force.
"""
from .lib import load, build  # noqa: F401
from .sim import OracleSim, from_config  # noqa: F401
