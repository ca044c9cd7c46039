"""B200-native DTR eviction-decision engine (arXiv 2006.09616, simrd V2 hot path).

Product path: libdtr.so (CUDA kernels for sm_100a, C ABI in include/dtr.h) and
this thin ctypes binding. There is no CPU fallback: importing fails loudly if
the library is missing.
"""
from .binding import (lib, Runtime, DeviceBatch, AdversaryBatch, ADV_DTYPE, abl_id, DEALLOC, replay_batch, replay_batch_host, pack_logs, make_cells,
                      cell_dims, workspace_bytes, cta_class, DtrError, HEURISTICS, ENGINE_CTA, ENGINE_GRID, STATUS_NAMES,
                      TRACE_DTYPE, RESULT_DTYPE, CELL_DTYPE, EXPORTS)

__all__ = ["lib", "Runtime", "DeviceBatch", "AdversaryBatch", "ADV_DTYPE", "abl_id", "DEALLOC", "replay_batch", "replay_batch_host", "pack_logs", "make_cells",
           "cell_dims", "workspace_bytes", "cta_class", "DtrError", "HEURISTICS", "ENGINE_CTA", "ENGINE_GRID",
           "STATUS_NAMES", "TRACE_DTYPE", "RESULT_DTYPE", "CELL_DTYPE", "EXPORTS"]
