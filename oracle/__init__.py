"""CPU fp64 oracle for BA-Att — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product package never
does (tests/test_boundary.py checks it).
"""
from .ba_oracle import *  # noqa: F401,F403
