"""One config-2 cell on the CTA engine (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
h = int(sys.argv[1]) if len(sys.argv) > 1 else 0
pm = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = models.resnet32()
v = LogView(w)
b = P.DeviceBatch([w], [dict(log=0, budget=v.budget(pm), heuristic=h)], engine=P.ENGINE_CTA)
for _ in range(reps):
    b.run()
torch.cuda.synchronize()
print(b.result_rows()[0])
