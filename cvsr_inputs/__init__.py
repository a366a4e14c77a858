"""Seeded input generators shared by the CUDA path and the oracle.

Holds NONE of the method's arithmetic (no quantiser, syndrome, LLR or decoder):
only code construction (the parity-check matrices are inputs), the quantiser's
fp32 edge table (a parameter), synthetic AWGN quadratures and the workload
configurations.  See DESIGN.md "Boundary and independence".
"""
from . import awgn, codes, configs, quantiser  # noqa: F401
from ._native import build  # noqa: F401
