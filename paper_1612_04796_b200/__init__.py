"""B200-native (sm_100a, FP64) p-multigrid for nodal IP-DG Poisson problems on periodic
Cartesian grids — arXiv:1612.04796 (Stiller).  Thin ctypes binding over the C ABI in
include/pmg_dg.h; every step of the hot path runs in the CUDA kernels of libpmgdg.so.
PyTorch provides device memory and streams only.  There is no CPU fallback: if the
shared library is missing this import fails.
"""
from .binding import (DG, lib, PMGError, GLL, GL, OVL_NODES, OVL_REL, OVL_MAXREL,  # noqa: F401
                      dg_setup)

from .slab import SlabDG  # noqa: F401,E402

__all__ = ["DG", "SlabDG", "dg_setup", "PMGError", "GLL", "GL", "OVL_NODES", "OVL_REL", "OVL_MAXREL"]
