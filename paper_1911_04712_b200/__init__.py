"""B200-native DPD solvent step (Mirheo, arXiv:1911.04712).

The product is ``libdpd.so`` (CUDA for sm_100a behind the C-ABI in ``include/dpd.h``);
``capi`` is its ctypes binding with the same names.  See DESIGN.md.
"""
from .capi import DPD, DPDError, load  # noqa: F401
from . import capi  # noqa: F401
