import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models
h = int(sys.argv[1]) if len(sys.argv) > 1 else 0
w = models.linear(64)
b = P.DeviceBatch([w], [dict(log=0, budget=16, heuristic=h, thrash_kill=0)], engine=P.ENGINE_GRID)
b.run(); torch.cuda.synchronize()
print(h, b.result_rows()[0])
