"""Probe: grid-engine timing vs decision cap on the config-5s stress log."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
s = torch.cuda.current_stream()
if n > 0:
    w = models.random_dag(n, seed=0)
    v = LogView(w)
for h in ((0, 1, 2) if n > 0 else ()):
    for D in (1, 101, 1001, 3001):
        spec = [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=h, thrash_kill=16, max_decisions=D)]
        b = P.DeviceBatch([w], spec, engine=P.ENGINE_GRID)
        b.run(s); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); b.run(s); e1.record(s); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        r = b.result_rows()[0]
        print(f"h={h} D={D} ms={[round(t,2) for t in ts]} status={r['status']} dec={r['decisions']} rec={r['records_done']} "
              f"evals={r['cand_evals']} bytes={r['score_bytes']}", flush=True)
        del b
# CTA engine per-cell timing on config 2
w = models.resnet32()
v = LogView(w)
for h in (0, 1, 2, 3):
    for pm in (100, 400, 1000):
        spec = [dict(log=0, budget=v.budget(pm), heuristic=h)]
        b = P.DeviceBatch([w], spec, engine=P.ENGINE_CTA)
        b.run(s); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); b.run(s); e1.record(s); torch.cuda.synchronize()
        r = b.result_rows()[0]
        ms = e0.elapsed_time(e1)
        print(f"cta h={h} pm={pm} ms={ms:.3f} dec={r['decisions']} evals={r['cand_evals']} rec={r['records_done']} "
              f"us/dec={1e3*ms/max(1,int(r['decisions'])):.2f} us/rec={1e3*ms/max(1,int(r['records_done'])):.3f}")
