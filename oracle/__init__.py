"""CPU float64 oracle for Tactic decode -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this package.  The product package never does.
"""
from . import tactic_oracle  # noqa: F401
from .tactic_oracle import *  # noqa: F401,F403
