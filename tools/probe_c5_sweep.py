"""The config-5 sweep (bench's headline step) once with the static cost estimate and
once ordered by the measured cell times: step time, and the slowest cells."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2006_09616_b200 import sweep
logs, views, cells = bench.workload_c5()
costs = None
out = open(os.environ.get("OUT", "gpurun_out/c5_sweep.jsonl"), "a")
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    rs = sweep.RankSweep(logs, views, cells, costs=costs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); rs.run(); e1.record(); torch.cuda.synchronize()
    rows = sweep.order_by_cell(np.concatenate([b.result_rows() for b in rs.batches]))
    ms = e0.elapsed_time(e1)
    costs = {int(r["cell_id"]): int(r["wall_ns"]) for r in rows}
    dec = int(rows["decisions"].sum())
    print(f"run {it}: {ms:.0f} ms, {dec} decisions, {dec / ms * 1e3:.0f} decisions/s", flush=True)
    grp = {}
    for c, r in zip(cells, rows):
        k = (bench.C5_MODELS[c["log"]], [h for h, v in bench.HEUR_IDS.items() if v == c["heuristic"]][0])
        g = grp.setdefault(k, [0, 0, 0])
        g[0] = max(g[0], int(r["wall_ns"]) / 1e6); g[1] += int(r["wall_ns"]) / 1e6; g[2] += int(r["decisions"])
    for k, g in sorted(grp.items(), key=lambda x: -x[1][0])[:12]:
        print(f"   {k[0]:12s} {k[1]:7s} max cell {g[0]:9.1f} ms  sum {g[1]:10.1f} ms  decisions {g[2]}", flush=True)
    out.write(json.dumps({"run": it, "ms": ms, "decisions": dec, "wall_ns": [int(x) for x in rows["wall_ns"]],
                          "dec": [int(x) for x in rows["decisions"]], "status": [int(x) for x in rows["status"]]}) + "\n")
    out.flush()
    del rs
