"""B200-native HeteGen heterogeneous offloaded linear (arXiv 2403.01164).

The product is the C-ABI library libhg.so (include/hg.h); `hg` is its thin
ctypes binding.  See DESIGN.md.
"""
from . import hg  # noqa: F401  (raises ImportError if libhg.so is missing: no fallback)
from .hg import Context, HgError, hg_plan, make_rates  # noqa: F401
