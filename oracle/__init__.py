"""fp64 CPU oracle for arXiv 1505.02100 (Algorithm 1) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  See oracle/oracle.py.
"""
from .oracle import *  # noqa: F401,F403
from .oracle import build, lib, plugin, psi, psi_literal, step1, zscore  # noqa: F401
