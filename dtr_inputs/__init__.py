"""Seeded synthetic inputs for DTR replays (shared by the oracle and the CUDA path).

Holds no arithmetic of the method: only the log encoding (logfmt) and workload
generators (models) whose shapes follow the paper's workloads.
"""
from .logfmt import (LogBuilder, LogView, assemble, MAGIC, HEADER_WORDS, OP_MAKE, OP_GET,
                     OP_RELEASE, OP_REMAT, OP_ENSURE, OP_DEBUG_EVICT, OP_SHIFT, ID_MASK)
from . import models
