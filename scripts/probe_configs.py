"""Timing of config 5 (900-cell sweep) and config 4 (long-log single runs) on one GPU."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_09616_b200 as P
from paper_2006_09616_b200 import sweep
from dtr_inputs import models, LogView
what = sys.argv[1] if len(sys.argv) > 1 else "both"
if what in ("both", "c5"):
    t0 = time.time()
    logs = [models.CONFIG_MODELS[m]() for m in ("resnet32", "densenet100", "unet", "lstm", "treelstm", "transformer")]
    views = [LogView(w) for w in logs]
    print("gen", round(time.time() - t0, 1), [v.n for v in views], flush=True)
    cells = sweep.make_cells(views, models.sweep_permilles(30), ["dtr", "dtr_eq", "lru", "size", "msps"])
    shard = sweep.shard(cells, views, 1)[0]
    rs = sweep.RankSweep(logs, views, shard)
    for b in rs.batches:
        print("batch", b.engine, b.n_cells, b.ws_bytes >> 20, "MiB", flush=True)
    rs.run(); torch.cuda.synchronize()
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); rs.run(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        rows = np.concatenate([b.result_rows() for b in rs.batches])
        print(f"config5 900 cells: {ms:.1f} ms -> {900/ms*1e3:.0f} runs/s, decisions {int(rows['decisions'].sum())} "
              f"-> {rows['decisions'].sum()/ms*1e3/1e6:.2f} M dec/s; statuses {np.bincount(rows['status'])}", flush=True)
    # per-model time (one model at a time)
    for li, v in enumerate(views):
        sub = [c for c in shard if c["log"] == li]
        b = P.DeviceBatch(logs, sub, engine=P.ENGINE_CTA)
        b.run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
        r = b.result_rows()
        print(f"  model {li} n={v.n}: {len(sub)} cells {e0.elapsed_time(e1):.1f} ms, decisions {int(r['decisions'].sum())}, "
              f"max cell decisions {int(r['decisions'].max())}", flush=True)
if what in ("both", "c4"):
    for name, gen in (("lstm T=4096", lambda: models.lstm(T=4096, layers=2)),
                      ("transformer L=96", lambda: models.transformer(layers=96))):
        t0 = time.time(); w = gen(); v = LogView(w)
        print(name, "n", v.n, "ops", v.n_ops, "gen", round(time.time() - t0, 1), flush=True)
        B = v.peak_total * 100000 // v.n
        for h in (0, 1):
            for eng in (P.ENGINE_GRID, P.ENGINE_CTA):
                b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=h)], engine=eng)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
                r = b.result_rows()[0]
                print(f"  h={h} eng={eng} B={B}: {e0.elapsed_time(e1):.0f} ms status={r['status']} dec={r['decisions']} "
                      f"remats={r['remats']} evals/dec={int(r['cand_evals'])/max(1,int(r['decisions'])):.0f}", flush=True)
