"""Host logic of the multi-GPU sweep on CPU: deterministic LPT sharding and the
row-table all_gather + reorder, exercised with a world_size-2 gloo group."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from dtr_inputs import LogView, models


def _views():
    return [LogView(models.resnet32()), LogView(models.unet()), LogView(models.linear(64))]


def test_shard_deterministic_complete_balanced():
    from paper_2006_09616_b200 import sweep
    views = _views()
    cells = sweep.make_cells(views, models.sweep_permilles(30), ["dtr", "dtr_eq", "lru", "size", "msps"])
    assert len(cells) == 3 * 30 * 5
    for ws in (1, 2, 4, 8):
        a = sweep.shard(cells, views, ws)
        b = sweep.shard(cells, views, ws)
        assert [[c["cell_id"] for c in s] for s in a] == [[c["cell_id"] for c in s] for s in b]
        ids = sorted(c["cell_id"] for s in a for c in s)
        assert ids == list(range(len(cells)))
        loads = [sum(sweep.est_cost(c, views) for c in s) for s in a]
        assert max(loads) <= min(loads) + max(sweep.est_cost(c, views) for c in cells) + 1e-9


def test_budgets_and_engine_groups():
    from paper_2006_09616_b200 import sweep
    views = _views() + [LogView(models.random_dag(70000, seed=1))]
    cells = sweep.make_cells(views, [100, 1000], ["dtr"])
    for c in cells:
        assert c["budget"] == views[c["log"]].peak_live * c["permille"] // 1000
    cta, grid = sweep.engine_groups(cells, views)
    assert all(views[c["log"]].n >= sweep.GRID_MIN_TENSORS for c in grid) and len(grid) == 2
    assert len(cta) == len(cells) - 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2006_09616_b200 import sweep
    from paper_2006_09616_b200.binding import RESULT_DTYPE
    views = _views()
    cells = sweep.make_cells(views, [200, 500, 800], ["dtr", "lru"])
    mine = sweep.shard(cells, views, ws)[rank]
    # stand-in rows (the device replay is tested on GPU): cell_id and a checksum
    rows = np.zeros(len(mine), dtype=RESULT_DTYPE)
    for i, c in enumerate(mine):
        rows[i]["cell_id"] = c["cell_id"]
        rows[i]["clock"] = 1000 + c["cell_id"]
        rows[i]["decisions"] = rank
    local = torch.from_numpy(rows.view(np.uint8).copy())
    counts = [len(s) for s in sweep.shard(cells, views, ws)]
    table = sweep.order_by_cell(sweep.gather_rows(local, counts, ws))
    out_q.put((rank, table["cell_id"].tolist(), table["clock"].tolist(), table["decisions"].tolist()))
    dist.destroy_process_group()


def test_gather_rows_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2006_09616_b200 import sweep
    views = _views()
    cells = sweep.make_cells(views, [200, 500, 800], ["dtr", "lru"])
    owner = {c["cell_id"]: r for r, s in enumerate(sweep.shard(cells, views, 2)) for c in s}
    for rank, ids, clocks, decs in res:
        assert ids == list(range(len(cells)))
        assert clocks == [1000 + i for i in ids]
        assert decs == [owner[i] for i in ids]
