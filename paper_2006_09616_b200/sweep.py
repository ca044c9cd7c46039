"""Budget x heuristic sweeps sharded over GPUs.

The paper's methodology (Fig. 2): every (op log, budget
ratio, heuristic) cell is an independent simulation.  Cells are assigned to
ranks by a deterministic longest-processing-time-first greedy on an estimated
cost; each rank replays its cells with the CUDA engines (one launch per
shared-memory class, CTA per simulation; logs too large for a CTA go to the
whole-GPU engine); then ONE collective -- all_gather_into_tensor of fixed-size
result tables over NCCL (NVLink 5 / NVSwitch) -- gives every rank the full
table, reordered by cell id.  There is no per-decision communication: a single
simulation does not shard.

Host logic only (argument marshalling and bookkeeping); every replay runs in
libdtr.so kernels.
"""
from __future__ import annotations

import numpy as np

from .binding import (DeviceBatch, RESULT_DTYPE, ENGINE_CTA, ENGINE_GRID, HEURISTICS, GRID_MIN_TENSORS,
                      cta_class)

# relative per-decision cost of a heuristic's score (MSPS walks closures)
HEUR_WEIGHT = {0: 3.0, 1: 3.0, 2: 1.0, 3: 1.0, 4: 6.0, 5: 1.5, 6: 1.0, 7: 8.0, 8: 8.0}


def make_cells(log_views, permilles, heuristics, thrash_kill=16, max_decisions=0):
    """Cells of a sweep: every log x budget permille x heuristic (names or ids).
    Returns a list of dicts {cell_id, log, permille, budget, heuristic, ...}."""
    cells = []
    for li, v in enumerate(log_views):
        for h in heuristics:
            hid = HEURISTICS[h] if isinstance(h, str) else int(h)
            for pm in permilles:
                cells.append(dict(cell_id=len(cells), log=li, permille=int(pm), budget=v.budget(pm),
                                  heuristic=hid, thrash_kill=thrash_kill, max_decisions=max_decisions))
    return cells


def est_cost(cell, log_views, costs=None):
    """Estimated cost of a cell: its MEASURED device time (costs[cell_id], e.g. the
    wall_ns of a previous run's row) when given, else a static guess."""
    if costs is not None and cell["cell_id"] in costs:
        return float(costs[cell["cell_id"]])
    v = log_views[cell["log"]]
    pm = max(int(cell.get("permille", 1000)), 50)
    h = cell["heuristic"]
    w = HEUR_WEIGHT.get(h, 8.0 if h in (16, 17, 18, 19) else 3.0 if h in (20, 21, 22, 23) else 1.0)
    return v.n_ops * (1000.0 / pm) * w


def shard(cells, log_views, world_size, costs=None):
    """Deterministic LPT: sort by (estimated or measured) cost (desc, then cell id),
    give each cell to the least-loaded rank (ties -> lowest rank). Returns per-rank lists."""
    order = sorted(cells, key=lambda c: (-est_cost(c, log_views, costs), c["cell_id"]))
    load = [0.0] * world_size
    out = [[] for _ in range(world_size)]
    for c in order:
        r = min(range(world_size), key=lambda k: (load[k], k))
        out[r].append(c)
        load[r] += est_cost(c, log_views, costs)
    for r in range(world_size):
        out[r].sort(key=lambda c: c["cell_id"])
    return out


def engine_groups(cells, log_views):
    """Split a rank's cells into the CTA-engine group and the grid-engine group."""
    cta = [c for c in cells if log_views[c["log"]].n < GRID_MIN_TENSORS]
    grid = [c for c in cells if log_views[c["log"]].n >= GRID_MIN_TENSORS]
    return cta, grid


class RankSweep:
    """The device side of one rank: its cells as (up to) two resident batches.

    CTA cells are grouped by shared-memory class (one launch each, the classes
    run concurrently) and, inside a class, ordered LONGEST FIRST by cost --
    measured device times when `costs` is given (sweep rows' wall_ns), else
    the static estimate: the hardware dispatches a launch's CTAs in order as
    SMs free up, so this is a longest-first work queue and the long cells
    never start in the last wave."""

    def __init__(self, logs, log_views, cells, device=None, costs=None):
        self.cells = cells
        cta, grid = engine_groups(cells, log_views)

        def key(c):
            v = log_views[c["log"]]
            return (cta_class(v.n, v.n_edges, c["heuristic"]), -est_cost(c, log_views, costs), c["cell_id"])
        cta.sort(key=key)
        grid.sort(key=lambda c: (-est_cost(c, log_views, costs), c["cell_id"]))
        self.order = cta + grid
        self.batches = []
        for group, eng in ((cta, ENGINE_CTA), (grid, ENGINE_GRID)):
            if group:
                self.batches.append(DeviceBatch(logs, group, engine=eng, device=device))

    def run(self, stream=None):
        for b in self.batches:
            b.run(stream)

    def rows_device(self):
        import torch
        return torch.cat([b.rows for b in self.batches]) if self.batches else None


def gather_rows(local_rows_u8, counts, world_size, group=None):
    """ONE all_gather_into_tensor of fixed-size row tables (each rank's padded to
    max(counts) rows).  counts[r] = rank r's number of cells -- every rank knows
    them from the deterministic shard(), so no collective is spent on them.
    Returns the concatenated table as a numpy structured array (valid rows only)."""
    import torch
    import torch.distributed as dist
    rb = RESULT_DTYPE.itemsize
    dev = local_rows_u8.device
    max_local = max(max(counts), 1)
    rank = dist.get_rank(group) if world_size > 1 else 0
    n_local = int(counts[rank])
    padded = torch.zeros(max_local * rb, dtype=torch.uint8, device=dev)
    if n_local:
        padded[: n_local * rb] = local_rows_u8[: n_local * rb]
    if world_size > 1:
        if dev.type == "cuda" and dist.get_backend(group) == "gloo":
            padded = padded.cpu()            # gloo gathers host tensors (CPU tests, world-2 GPU test)
        out = torch.empty(world_size * max_local * rb, dtype=torch.uint8, device=padded.device)
        dist.all_gather_into_tensor(out, padded, group=group)
    else:
        out = padded
    table = out.cpu().numpy().view(RESULT_DTYPE).reshape(world_size, max_local)
    return np.concatenate([table[r, : int(counts[r])] for r in range(world_size)])


def order_by_cell(rows):
    return rows[np.argsort(rows["cell_id"], kind="stable")]


def run_sweep(logs, log_views, cells, rank=0, world_size=1, device=None, group=None):
    """Replay every cell of a sweep across the process group; every rank returns
    the full table ordered by cell id."""
    import torch
    shards = shard(cells, log_views, world_size)
    mine = shards[rank]
    rs = RankSweep(logs, log_views, mine, device=device)
    rs.run()
    torch.cuda.synchronize()
    local = rs.rows_device()
    if local is None:
        local = torch.zeros(0, dtype=torch.uint8, device=device or "cuda")
    rows = gather_rows(local, [len(s) for s in shards], world_size, group)
    return order_by_cell(rows)
