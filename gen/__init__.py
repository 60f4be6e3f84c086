"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds *none* of the method's arithmetic: no D-ReLU, no degree
normalisers, no SpMM, no projections. It only draws CircuitNet-shaped graphs,
features, labels and parameters (SURVEY.md §8(d) recipe, restated in DESIGN.md
"Input recipe"), so both sides of every parity test start from identical arrays.
"""
from .circuit import (  # noqa: F401
    Design,
    disjoint_union,
    CONFIGS,
    make_design,
    make_config,
    make_params,
    make_c5_set,
    powerlaw_degrees,
)
