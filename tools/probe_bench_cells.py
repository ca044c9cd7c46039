"""Per-cell device time (wall_ns) of the bench's config-2 batch: which cells set the step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
import bench
logs, specs = bench.workload_c2(0)
b = P.DeviceBatch(logs, specs, engine=P.ENGINE_CTA)
for it in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
    print("launch ms", round(e0.elapsed_time(e1), 3))
r = b.result_rows()
for h in bench.C2_HEURS:
    idx = [i for i, s in enumerate(specs) if s["heuristic"] == bench.HEUR_IDS[h]]
    w = sorted(((int(r["wall_ns"][i]), int(r["decisions"][i]), i) for i in idx), reverse=True)[:3]
    print(h, [(round(a / 1e6, 3), d, i) for a, d, i in w])
