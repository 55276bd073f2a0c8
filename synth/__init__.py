"""Seeded synthetic instance generators shared by the oracle tests, the GPU tests and bench.py.

This module is plumbing: it builds problem data (A, b, l, u, f, incumbents) with the shapes of the
paper's QPLIB workloads (Table 1) as recipes in SURVEY.md §8(d)-1.
It holds none of MAPLE's arithmetic (no lattice, descent, rounding, check, filter or augmentation),
so importing it from both sides does not couple the oracle to the CUDA path.
"""
from .instances import (  # noqa: F401
    Instance,
    all_ones,
    assignment,
    c1,
    c2a,
    c2b,
    c3,
    c5,
    c4_batch,
    config,
    semi_assignment,
    random_small,
    partition_row,
    feasible_points,
)
