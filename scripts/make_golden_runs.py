"""Write expected full-length result rows for GPU parity tests, computed by the
CPU oracle ONLY (oracle/, plain C; no CUDA-path code is imported or run).

  python scripts/make_golden_runs.py run  OUT.jsonl  model:heur:permille ...   (one process per cell,
                                                      --timeout S per cell, --jobs J in parallel)
  python scripts/make_golden_runs.py one  model heur permille                  (worker: one JSON line)
  python scripts/make_golden_runs.py pack OUT.json IN.jsonl ...                (golden file for tests/)

Logs are the seeded synthetic generators of dtr_inputs (seed 0); budgets follow
reading C-16 (B = floor(peak_live * permille / 1000)); thrash_kill 16 (C-13)."""
import json
import os
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
FIELDS = ("status", "clock", "base", "decisions", "remats", "computations", "peak_M", "trace_hash", "records_done")


def gen(model):
    from dtr_inputs import models
    if model == "lstm4096":                    # config 4a: LSTM T=4096, 2 layers
        return models.lstm(T=4096, layers=2)
    if model == "transformer512":              # config 4b: Transformer, 512 layers, seq 256
        return models.transformer(layers=512)
    return models.CONFIG_MODELS[model]()


def one(model, heur, pm):
    from dtr_inputs import LogView
    from oracle import oracle as O
    w = gen(model)
    v = LogView(w)
    # "c4": config 4's budget rule B = peak_total * 1e5 / n (a ~1e5-tensor pool);
    # otherwise a permille of peak_live (reading C-16)
    B = v.peak_total * 100000 // v.n if pm == "c4" else v.budget(int(pm))
    t0 = time.time()
    r, _ = O.replay(w, O.HEURISTICS[heur], B, thrash_kill=16)
    rec = dict(model=model, heuristic=heur, permille=pm if pm == "c4" else int(pm), budget=int(B), seed=0,
               thrash_kill=16,
               oracle_s=round(time.time() - t0, 3))
    rec.update({f: int(r[f]) for f in FIELDS})
    print(json.dumps(rec), flush=True)


def run(out, cells, timeout, jobs):
    def go(c):
        m, h, pm = c.split(":")
        try:
            p = subprocess.run([sys.executable, __file__, "one", m, h, pm], capture_output=True, text=True,
                               timeout=timeout)
            line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else None
        except subprocess.TimeoutExpired:
            line = None
        if line:
            with open(out, "a") as f:
                f.write(line + "\n")
        print(c, "ok" if line else "timeout/fail", flush=True)
    with ThreadPoolExecutor(jobs) as ex:
        list(ex.map(go, cells))


if __name__ == "__main__":
    a = sys.argv[1:]
    if a[0] == "one":
        one(*a[1:4])
    elif a[0] == "run":
        timeout, jobs = 3600, max(1, (os.cpu_count() or 2) - 1)
        rest = []
        i = 2
        while i < len(a):
            if a[i] == "--timeout":
                timeout = float(a[i + 1]); i += 2
            elif a[i] == "--jobs":
                jobs = int(a[i + 1]); i += 2
            else:
                rest.append(a[i]); i += 1
        run(a[1], rest, timeout, jobs)
    elif a[0] == "pack":
        seen = {}
        for fn in a[2:]:
            for l in open(fn):
                if l.strip():
                    r = json.loads(l)
                    seen[(r["model"], r["heuristic"], str(r["permille"]))] = r
        rows = list(seen.values())
        rows.sort(key=lambda r: (r["model"], r["heuristic"], str(r["permille"]).zfill(6)))
        doc = {"citation": "Full-length simrd V2 runs (PAPER.md Doc A, P:213-373; heuristics P:96-111, "
                           "P:2286-2293, P:1261-1264) on the seeded synthetic config-5 logs (SURVEY.md 8(d)); "
                           "expected rows computed by oracle/ only (scripts/make_golden_runs.py).",
               "fields": list(FIELDS), "rows": rows}
        json.dump(doc, open(a[1], "w"), indent=1)
