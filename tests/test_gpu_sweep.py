"""The sharded sweep on one GPU (world_size 1): mixed shared-memory classes and
engines in one call, every row identical to the oracle's."""
import pytest

from dtr_inputs import LogView, models

pytestmark = pytest.mark.gpu
FIELDS = ("status", "records_done", "clock", "base", "decisions", "remats", "computations", "peak_M",
          "trace_hash")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_sweep_mixed_vs_oracle(torch_cuda, oracle_mod):
    from paper_2006_09616_b200 import sweep
    logs = [models.linear(64), models.resnet32(), models.unet(), models.densenet100(), models.transformer(layers=2)]
    views = [LogView(w) for w in logs]
    cells = sweep.make_cells(views, [150, 400, 700, 1000], ["dtr", "dtr_eq", "lru", "size", "msps"])
    rows = sweep.run_sweep(logs, views, cells)
    assert [int(r["cell_id"]) for r in rows] == [c["cell_id"] for c in cells]
    for c, r in zip(cells, rows):
        ref, _ = oracle_mod.replay(logs[c["log"]], c["heuristic"], c["budget"], thrash_kill=16)
        for f in FIELDS:
            assert int(r[f]) == int(ref[f]), (c, f)


def test_sweep_grid_group_vs_oracle(torch_cuda, oracle_mod):
    from paper_2006_09616_b200 import sweep
    logs = [models.random_dag(80000, seed=5), models.resnet32()]
    views = [LogView(w) for w in logs]
    cells = sweep.make_cells(views, [980], ["dtr", "lru"], max_decisions=40)
    rows = sweep.run_sweep(logs, views, cells)
    for c, r in zip(cells, rows):
        ref, _ = oracle_mod.replay(logs[c["log"]], c["heuristic"], c["budget"], thrash_kill=16,
                                   max_decisions=40)
        for f in FIELDS:
            assert int(r[f]) == int(ref[f]), (c, f)


def _w2_cells():
    from paper_2006_09616_b200 import sweep
    logs = [models.resnet32(), models.unet(), models.linear(64)]
    views = [LogView(w) for w in logs]
    return logs, views, sweep.make_cells(views, [150, 400, 700, 1000], ["dtr", "dtr_eq", "lru", "size", "msps"])


def _w2_worker(rank, ws, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    torch.cuda.set_device(0)
    from paper_2006_09616_b200 import sweep
    logs, views, cells = _w2_cells()
    rows = sweep.run_sweep(logs, views, cells, rank=rank, world_size=ws, device=0)
    rows["wall_ns"] = 0
    q.put((rank, rows.tobytes()))
    dist.destroy_process_group()


def test_sweep_world2_real_rows(torch_cuda, oracle_mod):
    """SURVEY 8(e) correctness check: two ranks (one process each, both on
    cuda:0, gloo for the one gather) replay their real LPT shards; the gathered
    table is byte-identical to the world-1 table and row-identical to the oracle."""
    import multiprocessing as mp
    import socket
    from paper_2006_09616_b200 import sweep
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_w2_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    logs, views, cells = _w2_cells()
    assert all(len(x) for x in sweep.shard(cells, views, 2))
    one = sweep.run_sweep(logs, views, cells)
    one["wall_ns"] = 0
    assert got[0] == got[1] == one.tobytes()
    for c, r in zip(cells, one):
        ref, _ = oracle_mod.replay(logs[c["log"]], c["heuristic"], c["budget"], thrash_kill=16)
        for f in FIELDS:
            assert int(r[f]) == int(ref[f]), (c, f)
