"""Time dtr_pool_argmin on the 1e6 stress pool for several heuristics (L2 flushed before each launch)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
w = models.random_dag(n, seed=0); v = LogView(w)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for h in (0, 1, 2, 3):
    b = P.DeviceBatch([w], [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=h, max_decisions=1000)], engine=P.ENGINE_GRID)
    b.run(); torch.cuda.synchronize()
    for l2 in (True, False):
        ts = []
        for _ in range(10):
            if l2: flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); o = b.pool_argmin(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        o = o.cpu().numpy()
        print(f"h={h} flush={l2} us median={sorted(ts)[5]:.1f} min={min(ts):.1f} id={o[2]} bytes={o[3]} evals={o[4]}")
