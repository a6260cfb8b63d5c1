"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This module holds ONLY problem parameters (BASELINE.json configs) and seeded
random-number generation.  It contains none of the method's arithmetic (no
basis, no operator, no smoother), so importing it from both `oracle/` and the
product/test side does not couple the two implementations.
"""
from .configs import CONFIGS, get_config, OverlapSpec  # noqa: F401
from .generators import uniform_zero_mean, uniform_vector  # noqa: F401
