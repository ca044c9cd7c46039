"""Per-decision cost on the LSTM log (config 5), CTA vs grid engine, capped."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
w = models.lstm(); v = LogView(w)
for h in (0, 1, 2, 3, 4):
    for pm in (300, 1000):
        for eng in (P.ENGINE_CTA, P.ENGINE_GRID):
            D = 300 if h == 4 else 3000
            res = []
            for cap in (D // 3, D):
                b = P.DeviceBatch([w], [dict(log=0, budget=v.budget(pm), heuristic=h, max_decisions=cap)], engine=eng)
                b.run(); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
                r = b.result_rows()[0]
                res.append((e0.elapsed_time(e1), int(r["decisions"]), int(r["records_done"]), int(r["cand_evals"])))
            (t0, d0, r0, c0), (t1, d1, r1, c1) = res
            print(f"h={h} pm={pm} eng={eng}: {1e3*(t1-t0)/max(1,d1-d0):.1f} us/decision (pool~{(c1-c0)/max(1,d1-d0):.0f}), "
                  f"prefix {t0:.1f} ms for {r0} records", flush=True)
