"""Setup + dtr_pool_argmin timing at the 4e6 stress point (exceeds L2)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000000
t0 = time.time(); w = models.random_dag(n, seed=0, cost_max=60); v = LogView(w); t1 = time.time()
b = P.DeviceBatch([w], [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=0, max_decisions=int(sys.argv[2]) if len(sys.argv) > 2 else 1000)], engine=P.ENGINE_GRID)
torch.cuda.synchronize(); t2 = time.time()
b.run(); torch.cuda.synchronize(); t3 = time.time()
print(f"gen {t1-t0:.1f}s upload {t2-t1:.1f}s replay {t3-t2:.1f}s row {b.result_rows()[0]}")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); o = b.pool_argmin(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1000)
o = o.cpu().numpy()
print(f"us median={sorted(ts)[5]:.1f} min={min(ts):.1f} bytes={o[3]} evals={o[4]} GB/s={o[3]/sorted(ts)[5]/1e3:.0f}")
