"""Config 5 uncapped, one (model, heuristic) group of 30 budget cells per launch:
group time (= its slowest cell) and per-cell decisions/status."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
NAMES = ("resnet32", "densenet100", "unet", "lstm", "treelstm", "transformer")
HS = sys.argv[1].split(",") if len(sys.argv) > 1 else ["size", "lru", "dtr", "dtr_eq", "msps"]
MS = sys.argv[2].split(",") if len(sys.argv) > 2 else list(NAMES)
out = open(os.environ.get("OUT", "gpurun_out/c5_groups.jsonl"), "a")
logs = {m: models.CONFIG_MODELS[m]() for m in MS}
for h in HS:
    for m in MS:
        w = logs[m]; v = LogView(w)
        specs = [dict(log=0, budget=v.budget(pm), heuristic=P.HEURISTICS[h], thrash_kill=16)
                 for pm in models.sweep_permilles(30)]
        b = P.DeviceBatch([w], specs, engine=P.ENGINE_CTA)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
        r = b.result_rows()
        rec = dict(model=m, n=v.n, h=h, ms=e0.elapsed_time(e1), dec=[int(x) for x in r["decisions"]],
                   status=[int(x) for x in r["status"]], evals=[int(x) for x in r["cand_evals"]])
        out.write(json.dumps(rec) + "\n"); out.flush()
        print(m, h, f"{rec['ms']:.1f} ms", "max dec", max(rec["dec"]), "sum", sum(rec["dec"]), flush=True)
        del b
