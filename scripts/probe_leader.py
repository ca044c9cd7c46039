"""Grid-engine leader cost per log record vs grid size (env DTR_GRID_BLOCKS)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
w = models.random_dag(n, seed=0)
v = LogView(w)
s = torch.cuda.current_stream()
for D in (1, 201):
    spec = [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=0, thrash_kill=16, max_decisions=D)]
    b = P.DeviceBatch([w], spec, engine=P.ENGINE_GRID)
    b.run(s); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); b.run(s); e1.record(s); torch.cuda.synchronize()
    r = b.result_rows()[0]
    ms = e0.elapsed_time(e1)
    print(f"blocks={os.environ.get('DTR_GRID_BLOCKS','auto')} n={n} D={D} ms={ms:.1f} rec={r['records_done']} "
          f"us/rec={1e3*ms/max(1,int(r['records_done'])):.3f} evals={r['cand_evals']}", flush=True)
