import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
dev = torch.device("cuda", 0)
what = sys.argv[1]
if what == "c4":
    T = int(sys.argv[2])
    w = models.lstm(T=T, layers=2); v = LogView(w)
    B = v.peak_total * 100000 // v.n
    for D in (1000, 10000, 50000):
        b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=0, max_decisions=D)], engine=P.ENGINE_GRID)
        t0 = time.time(); b.run(); torch.cuda.synchronize(); t = time.time() - t0
        r = b.result_rows()[0]
        print(f"T={T} n={v.n} D={D}: {t:.2f} s status={r['status']} dec={r['decisions']} rec={r['records_done']}/{v.n_ops} pool~{int(r['cand_evals'])/max(1,int(r['decisions'])):.0f}", flush=True)
elif what == "c5":
    t0 = time.time(); print(bench.config5(P, torch, dev, cap=int(sys.argv[2])), time.time() - t0, flush=True)
