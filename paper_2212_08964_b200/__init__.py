"""B200-native CSR SpMV under programmable load-balancing schedules (arXiv 2212.08964).

The compute path is liblb.so (include/lb.h, csrc/); this package is its thin binding.
"""
from .lb import (LIB_PATH, CsrMatrix, Comm, HostSpmv, InvalidCsr, LbError, SCHEDULES, declared_functions,  # noqa: F401
                 gather_slices, last_error, launch_count, lib, shard_bounds, shard_csr, spmv, version)
