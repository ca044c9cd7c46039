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
