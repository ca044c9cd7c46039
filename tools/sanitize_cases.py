"""Small invocations of every kernel of libdtr.so for compute-sanitizer
(memcheck / racecheck / synccheck): tools/sanitize.sh runs this under each tool.

  python tools/sanitize_cases.py {cta,cta_global,grid,pool_argmin,percall,adversary}
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2006_09616_b200 as P  # noqa: E402
from dtr_inputs import LogView, models  # noqa: E402


def run(case):
    if case == "cta":            # K6, state in shared memory: every config-5 heuristic incl. MSPS (K5, closure cache)
        w = models.resnet32()
        v = LogView(w)
        specs = [dict(log=0, budget=v.budget(pm), heuristic=P.HEURISTICS[h])
                 for h in ("dtr", "dtr_eq", "lru", "size", "msps", "dtr_full") for pm in (200, 600)]
        b = P.DeviceBatch([w], specs, engine=P.ENGINE_CTA)
        b.run()
    elif case == "cta_global":   # K6, state in the global workspace (stream pass + slow stack)
        w = models.transformer(layers=2)
        v = LogView(w)
        specs = [dict(log=0, budget=v.budget(300), heuristic=P.HEURISTICS[h], max_decisions=300)
                 for h in ("dtr", "dtr_eq", "msps")]
        b = P.DeviceBatch([w], specs, engine=P.ENGINE_CTA)
        b.run()
    elif case in ("grid", "pool_argmin"):   # K7 (+ K3+K4 alone)
        w = models.random_dag(70000, seed=1)
        v = LogView(w)
        for h in ("dtr", "dtr_eq"):
            b = P.DeviceBatch([w], [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=P.HEURISTICS[h],
                                         max_decisions=30)], engine=P.ENGINE_GRID)
            b.run()
            if case == "pool_argmin":
                b.pool_argmin()
    elif case == "percall":      # the per-call runtime (percall_engine)
        rt = P.Runtime(P.HEURISTICS["dtr"], budget=6)
        ids = []
        for i in range(12):
            rc, t = rt.compute(1, 1 + i % 3, ids[-2:])
            ids.append(t)
        rt.scores()
        rt.close()
    elif case == "adversary":    # K8
        ab = P.AdversaryBatch([dict(n=200, budget=8, heuristic=P.HEURISTICS[h]) for h in ("dtr", "lru", "msps")])
        ab.run()
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(case, "ok")


if __name__ == "__main__":
    run(sys.argv[1])
