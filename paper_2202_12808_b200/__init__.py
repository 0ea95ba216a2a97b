"""B200-native covariance-free EM (CoFEM, arXiv 2202.12808) hot path.

The product is the C-ABI library `libcofem.so` (include/cofem.h) built from
`csrc/*.cu` for sm_100a; `cofem.py` is its thin ctypes binding.  There is no CPU
fallback.  See DESIGN.md.
"""
from .cofem import (OP_CIRCCONV, OP_DCT2_MASKED, OP_DENSE, CofemError, Context, get_unique_id,  # noqa: F401
                    kernel_classes, lib, probe_split)
