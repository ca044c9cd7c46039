"""One grid-engine run on the config-5s stress log (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
D = int(sys.argv[2]) if len(sys.argv) > 2 else 32
w = models.random_dag(n, seed=0); v = LogView(w)
b = P.DeviceBatch([w], [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=0, max_decisions=D)], engine=P.ENGINE_GRID)
for _ in range(2):
    b.run()
torch.cuda.synchronize()
print(b.result_rows()[0])
