"""One config-5 cell on the CTA engine (for ncu): MODEL HEUR PERMILLE [MAX_DECISIONS] [REPS]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
m, h, pm = sys.argv[1], sys.argv[2], int(sys.argv[3])
cap = int(sys.argv[4]) if len(sys.argv) > 4 else 0
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
w = models.CONFIG_MODELS[m]()
v = LogView(w)
b = P.DeviceBatch([w], [dict(log=0, budget=v.budget(pm), heuristic=P.HEURISTICS[h], max_decisions=cap)],
                  engine=P.ENGINE_CTA)
for _ in range(reps):
    b.run()
torch.cuda.synchronize()
print(b.result_rows()[0])
