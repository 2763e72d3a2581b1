"""B200-native cuTAMP particle-optimisation hot path (arXiv 2411.11833).

The product is libtamp.so (C ABI in include/tamp.h, sm_100a kernels in csrc/); `tamp` is the thin
ctypes binding.  See DESIGN.md.
"""
from .tamp import TampContext, build_desc, decode_records, kernel_launches, lib_path, load, merge_records, plan_heuristic, TampError  # noqa: F401
