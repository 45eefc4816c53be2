"""B200-native CSR SpMV under programmable load-balancing schedules (arXiv 2212.08964).

The compute path is liblb.so (include/lb.h, csrc/); this package is its thin binding.
"""
from .lb import (CHUNKS_MAX, LIB_PATH, SCHEDULES, TILE_LENGTHS, Comm, CsrMatrix, HostSpmv,  # noqa: F401
                 InvalidCsr, LbError, PeerBuffer, declared_functions, exchange_schedule, gather_slices, last_error,
                 launch_count, lib, padded_rows, remap_cols_padded, shard_bounds, shard_csr, spmv, version,
                 y_checksum)
