"""Seeded synthetic input generators shared by the CUDA path's tests/bench and
the oracle's tests.  Holds none of the method's arithmetic."""
from .workloads import CONFIGS, Workload, make_qkv, constant_block_qkv  # noqa: F401
