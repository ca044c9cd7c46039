"""Replay the stress log to D decisions on the grid engine, then run dtr_pool_argmin (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
h = int(sys.argv[2]) if len(sys.argv) > 2 else 0
w = models.random_dag(n, seed=0, cost_max=200 if n <= 1300000 else 60); v = LogView(w)
b = P.DeviceBatch([w], [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=h, max_decisions=1000)], engine=P.ENGINE_GRID)
b.run(); torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(4):
    flush.zero_()
    o = b.pool_argmin()
torch.cuda.synchronize()
print(o.cpu().numpy())
