#!/usr/bin/env python
"""bench.py -- DTR eviction-decision throughput on B200 (arXiv 2006.09616, simrd V2).

Workload (BASELINE.json configs[4], "config5", the largest single-GPU
configuration): the full budget x heuristic sweep of the paper's
methodology (Fig. 2) -- 6 synthetic models {ResNet-32,
DenseNet-100, UNet, LSTM, TreeLSTM, Transformer} x 30 budget ratios
(0.1..1.0) x {h_DTR, h_DTR_eq, LRU, size, MSPS} = 900 independent simulations,
EVERY ONE RUN TO ITS END (ok, OOM, or the thrash kill of reading C-13; no
decision cap).  The 900 cells are sharded over the N ranks by LPT (STRONG
scaling: the sweep is fixed); one step = each rank replays its cells with the
CTA-per-simulation engine (one launch per shared-memory class, cells longest
first by their measured device time) + ONE all_gather of the result rows.

  value   = eviction decisions / s of the whole sweep (all ranks), device-timed
            (CUDA events on the launching stream, max over ranks), inputs
            resident in HBM, L2 flushed (256 MiB write) before every step.
  runs_per_sec = 900 / step time.
  e2e     = the same metric through dtr_replay_batch_host (the public host-buffer
            entry): pinned host logs + cells in, rows out, H2D/D2H and
            stream-ordered allocation inside the timed region.
  roofline: the CTA engine (the only kernel of the step): algorithmic score-pass
            bytes per step / step time vs MEASURED_PEAKS.json hbm_gbs, plus the
            critical cell's device time per decision (the step is a latency
            chain).
  roofline_large_pool(_4e6): K3+K4 alone (dtr_pool_argmin) over the ~1e6 / 4e6
            pool of the config-5s stress log, CUDA-event timed, L2 flushed.
  config2_sweep: the ResNet-32 sweep (120 cells, BASELINE configs[1]).
  config4: LSTM T=4096 (323 k tensors) and Transformer L=512 (162 k) single runs
            to completion on the whole-GPU engine, the oracle's rate beside.
  config5s: the first 10^4 decisions of the 1e6-tensor stress log on the
            whole-GPU engine, the oracle's rate beside.
  cpu_baseline: the CPU oracle (oracle/, plain C, unmodified) on the host cores:
            the first <= 4000 decisions of each of the 720 cells, process pool.

`--impl reference` times the oracle alone (the reference arm for this tier).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from dtr_inputs import LogView, models  # noqa: E402

METRIC = "eviction decisions/sec (pool score+argmin) and sweep runs/sec at 1/2/4/8 B200"
C5_MODELS = ("resnet32", "densenet100", "unet", "lstm", "treelstm", "transformer")
C5_HEURS = ("dtr", "dtr_eq", "lru", "size")      # the headline; MSPS: --msps (config5_msps)
C2_HEURS = ("dtr", "dtr_eq", "lru", "size")
HEUR_IDS = {"dtr": 0, "dtr_eq": 1, "lru": 2, "size": 3, "msps": 4, "local": 5, "random": 6}
C5_WORKLOAD = ("config5 (h_DTR, h_DTR_eq, LRU, size): 6 models {resnet32,densenet100,unet,lstm,treelstm,transformer} "
               "x 30 budget ratios x 4 heuristics = 720 cells, every cell run to its end (no decision cap); the "
               "180 MSPS cells of the 900-cell sweep are timed separately (--msps, config5_msps)")
ORACLE_CAP = 4000   # cpu_baseline / reference arm: the first <= ORACLE_CAP decisions of each cell


def workload_c5(heurs=C5_HEURS):
    """config 5: the budget x heuristic sweep (seed-0 logs), uncapped."""
    logs = [models.CONFIG_MODELS[m]() for m in C5_MODELS]
    views = [LogView(w) for w in logs]
    cells = []                      # = sweep.make_cells (the reference arm does not import the product)
    for li, v in enumerate(views):
        for h in heurs:
            for pm in models.sweep_permilles(30):
                cells.append(dict(cell_id=len(cells), log=li, permille=pm, budget=v.budget(pm),
                                  heuristic=HEUR_IDS[h], thrash_kill=16, max_decisions=0))
    return logs, views, cells


def workload_c2(rank: int = 0):
    """config 2: ResNet-32-shaped log (seed = rank) x 30 permilles x 4 heuristics."""
    w = models.resnet32(seed=rank)
    v = LogView(w)
    specs = []
    for h in C2_HEURS:
        for pm in models.sweep_permilles(30):
            specs.append(dict(log=0, budget=v.budget(pm), heuristic=HEUR_IDS[h], thrash_kill=16,
                              cell_id=len(specs)))
    return [w], specs


# ---------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,utilization.gpu,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 10]
        load = [r for r in rows if _num(r[3]) and _num(r[3]) > 0] or rows
        sm = [_num(r[1]) for r in load if _num(r[1])]
        mx = [_num(r[2]) for r in rows if _num(r[2])]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in load:
            for k, nm in enumerate(names):
                if r[6 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(load)}


def _num(x):
    try:
        return float(x)
    except Exception:
        return None


# ---------------------------------------------------------------------------- cpu oracle

def _oracle_cell(args):
    words, h, budget, kill, cap = args
    from oracle import oracle as O
    t0 = time.perf_counter()
    r, _ = O.replay(words, h, budget, thrash_kill=kill, max_decisions=cap)
    return int(r["decisions"]), time.perf_counter() - t0


def _noop(_):
    return 0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_pass(jobs, pool):
    """One pass of the oracle over `jobs` on the pool: (decisions, wall s, summed per-cell s)."""
    t0 = time.perf_counter()
    dec, cpu = 0, 0.0
    for d, t in pool.imap_unordered(_oracle_cell, jobs, chunksize=1):
        dec += d
        cpu += t
    return dec, time.perf_counter() - t0, cpu


def oracle_jobs(logs, cells, cap=ORACLE_CAP):
    # longest logs first so the pool's tail is short
    order = sorted(cells, key=lambda c: -len(logs[c["log"]]))
    return [(logs[c["log"]], c["heuristic"], c["budget"], c.get("thrash_kill", 16), cap) for c in order]


def cpu_baseline(logs, cells, cores, pool=None):
    """The oracle, unmodified, on the host cores: the first <= ORACLE_CAP decisions
    of each config-5 cell (a bounded sample of the same workload), process pool
    started outside the timed sample."""
    import multiprocessing as mp
    from oracle import oracle as O
    O.build()
    jobs = oracle_jobs(logs, cells)
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(cores)
        pool.map(_noop, range(cores))
    try:
        dec, wall, cpu = oracle_pass(jobs, pool)
    finally:
        if own:
            pool.close()
            pool.join()
    return {"value": dec / wall, "unit": "decisions/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "single_thread_decisions_per_s": dec / cpu,
            "sample": f"the first <= {ORACLE_CAP} decisions of each of the {len(cells)} config-5 cells "
                      f"({dec} decisions), {cores}-process pool, {wall:.2f} s wall; single_thread = "
                      f"decisions / summed per-cell steady-clock time"}


# ---------------------------------------------------------------------------- main

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    logs, views, cells = workload_c5()
    cores = host_cores()
    import multiprocessing as mp
    from oracle import oracle as O
    O.build()
    jobs = oracle_jobs(logs, cells)
    vals = []
    with mp.get_context("fork").Pool(cores) as pool:      # one pool for the run, started before timing
        pool.map(_noop, range(cores))
        for i in range(args.warmup + args.steps):
            dec, wall, cpu = oracle_pass(jobs, pool)
            if i >= args.warmup:
                vals.append((dec, wall, cpu))
    dec = sum(v[0] for v in vals)
    wall = sum(v[1] for v in vals)
    cpu = sum(v[2] for v in vals)
    value = dec / wall
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "decisions/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "config": {"workload": C5_WORKLOAD, "cells": len(cells),
                       "sample": f"each step: the first <= {ORACLE_CAP} decisions of every cell"},
            "cpu_baseline": {"value": value, "unit": "decisions/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(), "single_thread_decisions_per_s": dec / cpu,
                             "sample": f"per step the first <= {ORACLE_CAP} decisions of each of the "
                                       f"{len(cells)} config-5 cells ({dec // args.steps} decisions), "
                                       f"{cores}-process pool"},
            "e2e": {"value": value, "unit": "decisions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-large-pool", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--large-n", type=int, default=1000000)
    ap.add_argument("--large-n2", type=int, default=4000000, help="second large-pool point (0 = skip)")
    ap.add_argument("--no-extra", action="store_true", help="skip the config-2 / config-4 / config-5s extras")
    ap.add_argument("--msps", action="store_true",
                    help="also replay the 180 MSPS cells of the config-5 sweep once (config5_msps; minutes)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2006_09616_b200 import sweep

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2006_09616_b200 as P

    logs, views, cells = workload_c5()
    n_cells = len(cells)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def build(costs):
        shards = sweep.shard(cells, views, ws, costs)
        return shards, sweep.RankSweep(logs, views, shards[rank], device=local, costs=costs)

    def step(rs, counts):
        rs.run(stream)
        local_rows = rs.rows_device()
        if local_rows is None:
            local_rows = torch.zeros(0, dtype=torch.uint8, device=dev)
        return sweep.gather_rows(local_rows, counts, ws)          # the one collective (N > 1)

    # warm-up 1: static cost estimate; its rows' device times (wall_ns, every
    # rank has every row after the gather) become the measured costs that shard
    # the sweep (LPT) and order each rank's cells longest first
    shards, rs = build(None)
    rows = step(rs, [len(x) for x in shards])
    costs = {int(r["cell_id"]): int(r["wall_ns"]) for r in rows}
    del rs
    shards, rs = build(costs)
    counts = [len(x) for x in shards]
    for _ in range(max(args.warmup - 1, 0)):
        rows = step(rs, counts)
    torch.cuda.synchronize()
    decisions_all = int(rows["decisions"].sum())
    score_bytes_rank = int(sum(int(b.result_rows()["score_bytes"].sum()) for b in rs.batches))
    # the dominant kernel: cta_engine_g, the launch of the cells whose state stays in global memory
    # (shared-memory class 2; ~99.6 % of the step in the ncu launch list)
    g_bytes = 0
    for b in rs.batches:
        if b.engine != P.ENGINE_CTA:
            continue
        br = b.result_rows()
        for k, sp in enumerate(b.specs):
            v = views[sp["log"]]
            if P.cta_class(v.n, v.n_edges, sp["heuristic"]) == 2:
                g_bytes += int(br["score_bytes"][k])
    crit = rows[int(np.argmax(rows["wall_ns"]))]
    launches_per_step = sum(b.launches_per_run() for b in rs.batches)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        rows = step(rs, counts)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    wall = time.perf_counter() - w0
    clocks = sampler.stop()
    assert int(rows["decisions"].sum()) == decisions_all and len(rows) == n_cells
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_rank = sum(step_ms) / 1e3
    if ws > 1:
        t = torch.tensor([t_rank], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    else:
        t_max = t_rank
    value = decisions_all * args.steps / t_max
    runs_per_sec = n_cells * args.steps / t_max

    # ---- e2e: this rank's shard through the public host-buffer entry (pinned host memory)
    import ctypes as C
    e2e_parts = []
    for b in rs.batches:
        words, offs = P.pack_logs(logs)
        hc, _ = P.make_cells(offs, b.specs)
        e2e_parts.append((torch.from_numpy(words.view(np.int32)).pin_memory(), len(words),
                          torch.from_numpy(hc.view(np.uint8)).pin_memory(), len(b.specs), b.engine,
                          torch.empty(len(b.specs) * P.RESULT_DTYPE.itemsize, dtype=torch.uint8).pin_memory()))

    def e2e_step():
        for hw, nw, hc, nc, eng, hr in e2e_parts:
            rc = P.lib.dtr_replay_batch_host(C.c_void_p(hw.data_ptr()), nw, C.c_void_p(hc.data_ptr()), nc, eng,
                                             C.c_void_p(hr.data_ptr()), None, 0, C.c_void_p(stream.cuda_stream))
            assert rc == 0, rc

    # the device path is warm (same kernels, same cells): one timed end-to-end step
    e2e_steps = 1
    e_s = 0.0
    for i in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        e_s += time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_s = float(t.item())
    e2e_dec = sum(int(hr.numpy().view(P.RESULT_DTYPE)["decisions"].sum()) for *_, hr in e2e_parts)
    assert e2e_dec == sum(int(b.result_rows()["decisions"].sum()) for b in rs.batches)
    e2e_value = decisions_all * e2e_steps / e_s
    h2d = sum(hw.numel() * 4 + hc.numel() for hw, _, hc, *_ in e2e_parts)
    d2h = sum(hr.numel() for *_, hr in e2e_parts)

    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak, peak_src = float(peaks["hbm_gbs"]), "measured"
    except Exception:
        hbm_peak, peak_src = 6650.0, "fallback"
    kern_s = t_rank / args.steps
    sm_hz = (clocks.get("sm_mhz") or 1965.0) * 1e6
    roof = {"bound": "hbm", "achieved": g_bytes / kern_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": g_bytes / kern_s / 1e9 / hbm_peak, "traffic": None, "peak_source": peak_src,
            "kernel": "cta_engine_g (global-state cells; the classes run concurrently, so its launch spans the step)",
            "algorithmic_bytes_per_launch": g_bytes, "algorithmic_bytes_per_step_all_classes": score_bytes_rank,
            "critical_cell": {"cell_id": int(crit["cell_id"]), "decisions": int(crit["decisions"]),
                              "device_ms": int(crit["wall_ns"]) / 1e6,
                              "us_per_decision": int(crit["wall_ns"]) / 1e3 / max(1, int(crit["decisions"])),
                              "cycles_per_decision": int(crit["wall_ns"]) * 1e-9 * sm_hz / max(1, int(crit["decisions"]))},
            "note": "the step is the longest cell's sequential decision chain (state in shared memory / L2); "
                    "HBM is not its bound -- see critical_cell and DESIGN.md 6"}
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(traffic_file):
        try:
            tf = json.load(open(traffic_file))
            roof["traffic"] = tf.get("cta_engine_g_config5")
            roof["traffic_critical_cell_20k_decisions"] = tf.get("cta_engine_g_lstm_dtr_eq_20k")
        except Exception:
            pass

    out = {"metric": METRIC, "value": value, "unit": "decisions/s", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
           "config": {"workload": C5_WORKLOAD, "cells": n_cells, "decisions_per_step": decisions_all,
                      "engine": "cta (one CTA per simulation), cells longest first by measured device time",
                      "l2": "flushed (256 MiB write) before each step",
                      "parallelism": f"sweep sharded over {ws} rank(s) (LPT on measured cell times), "
                                     f"one all_gather of the rows"},
           "runs_per_sec": runs_per_sec,
           "e2e": {"value": e2e_value, "unit": "decisions/s", "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "steps": e2e_steps},
           "gpu_launches": launches_per_step * args.steps,
           "roofline": roof,
           "clocks": clocks,
           "wall_s_timed": wall}

    if rank == 0 and not args.no_large_pool:
        out["roofline_large_pool"] = large_pool(P, torch, dev, args.large_n, hbm_peak, peak_src)
        if args.large_n2:   # the point that exceeds the 126 MB L2
            out["roofline_large_pool_4e6"] = large_pool(P, torch, dev, args.large_n2, hbm_peak, peak_src)
    if rank == 0 and ws == 1 and not args.no_extra:
        out["config2_sweep"] = config2(P, torch, dev, flush)
        out["config4"] = config4(P, torch, dev, not args.no_cpu)
        out["config5s"] = config5s(P, torch, dev, not args.no_cpu)
    if rank == 0 and ws == 1 and args.msps:
        out["config5_msps"] = config5_msps(P, torch, dev)
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(logs, cells, host_cores())
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _oracle_rate(words, h, budget, cap):
    from oracle import oracle as O
    O.build()
    t0 = time.perf_counter()
    r, _ = O.replay(words, h, budget, thrash_kill=16, max_decisions=cap)
    dt = time.perf_counter() - t0
    return {"decisions": int(r["decisions"]), "s": dt, "decisions_per_s": int(r["decisions"]) / dt,
            "kind": "oracle, one host thread", "sample": f"the first {int(r['decisions'])} decisions"}


def config2(P, torch, dev, flush, steps=20):
    """Config 2 (BASELINE configs[1]): the 120-cell ResNet-32 sweep, one CTA-engine launch."""
    logs, specs = workload_c2(0)
    b = P.DeviceBatch(logs, specs, engine=P.ENGINE_CTA)
    s = torch.cuda.current_stream(dev)
    for _ in range(3):
        b.run(s)
    ts = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        b.run(s)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    r = b.result_rows()
    dec = int(r["decisions"].sum())
    ms = sum(ts) / len(ts)
    return {"workload": "config2: resnet32-shaped log x 30 budget ratios x {h_DTR,h_DTR_eq,LRU,size} (120 cells)",
            "ms_per_step": ms, "decisions_per_step": dec, "decisions_per_s": dec / ms * 1e3,
            "runs_per_s": len(specs) / ms * 1e3}


def config4(P, torch, dev, with_oracle=True):
    """Config 4: long logs, single-run latency on the whole-GPU engine, each run
    to completion: LSTM T=4096 x 2 layers (323 k tensors) and Transformer L=512
    (162 k tensors, seq 256), B = peak_total * 1e5 / n (a ~1e5-tensor
    pool), h_DTR and h_DTR_eq; the oracle's single-thread rate on
    the first 300 decisions of each beside."""
    res = {}
    for name, w in (("lstm_T4096", models.lstm(T=4096, layers=2)), ("transformer_L512", models.transformer(layers=512))):
        v = LogView(w)
        B = v.peak_total * 100000 // v.n
        ent = {"workload": f"{name}: n={v.n} tensors, {v.n_ops} records, B=peak_total*1e5/n, run to completion"}
        for h, hn in ((0, "h_DTR"), (1, "h_DTR_eq")):
            b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=h, thrash_kill=16)], engine=P.ENGINE_GRID)
            s = torch.cuda.current_stream(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            b.run(s)
            e1.record(s)
            torch.cuda.synchronize()
            r = b.result_rows()[0]
            ms = e0.elapsed_time(e1)
            ent[hn] = {"ms": ms, "status": int(r["status"]), "records_done": int(r["records_done"]),
                       "decisions": int(r["decisions"]), "remats": int(r["remats"]),
                       "decisions_per_s": int(r["decisions"]) / ms * 1e3,
                       "mean_pool": int(r["cand_evals"]) / max(1, int(r["decisions"]))}
            if with_oracle:
                ent[hn]["oracle"] = _oracle_rate(w, h, B, 300)
            del b
        res[name] = ent
    return res


def config5_msps(P, torch, dev):
    """The 180 MSPS cells of the config-5 sweep (6 models x 30 budget ratios), each
    run to its end, in one replay (CTA engine, longest first by the static
    estimate); device time, decisions, and the slowest cell per model."""
    from paper_2006_09616_b200 import sweep
    logs, views, cells = workload_c5(("msps",))
    rs = sweep.RankSweep(logs, views, cells, device=dev.index)
    s = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    rs.run(s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    rows = np.concatenate([b.result_rows() for b in rs.batches])
    by = {}
    for r in rows:
        m = C5_MODELS[cells[int(r["cell_id"])]["log"]]
        by[m] = max(by.get(m, 0.0), int(r["wall_ns"]) / 1e6)
    dec = int(rows["decisions"].sum())
    return {"workload": "config5 MSPS: 6 models x 30 budget ratios = 180 cells, every cell run to its end",
            "ms": ms, "decisions": dec, "decisions_per_s": dec / ms * 1e3, "runs_per_s": len(cells) / ms * 1e3,
            "slowest_cell_ms_by_model": by}


def config5s(P, torch, dev, with_oracle=True, D=10000):
    """Config 5s: the 1e6-tensor random locality DAG, B = 0.98 * peak_total (a ~1e6
    pool at the first decision): the first D decisions on the whole-GPU engine
    (h_DTR), CUDA-event timed; the oracle's single-thread rate on its first 100."""
    w = models.random_dag(1000000, seed=0, cost_max=200)
    v = LogView(w)
    B = v.peak_total * 98 // 100
    b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=0, thrash_kill=16, max_decisions=D)],
                      engine=P.ENGINE_GRID)
    s = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    b.run(s)
    e1.record(s)
    torch.cuda.synchronize()
    r = b.result_rows()[0]
    ms = e0.elapsed_time(e1)
    out = {"workload": f"random locality DAG n={v.n}, B=0.98*peak_total, first {D} decisions, h_DTR",
           "ms": ms, "decisions": int(r["decisions"]), "decisions_per_s": int(r["decisions"]) / ms * 1e3,
           "mean_pool": int(r["cand_evals"]) / max(1, int(r["decisions"])), "status": int(r["status"])}
    if with_oracle:
        out["oracle"] = _oracle_rate(w, 0, B, 100)
    return out


def large_pool(P, torch, dev, n, hbm_peak, peak_src, D=1000, reps=20):
    """K3+K4 alone at a ~n pool: replay the config-5s stress log on the grid engine
    up to its D-th eviction decision (h_DTR), then time dtr_pool_argmin -- the
    score pass + exact argmin over the resident pool -- with CUDA events, L2
    flushed (256 MiB write) before every launch."""
    # cost U[1,200] keeps base <= 2^27 up to ~1.3e6 tensors; beyond, U[1,60]
    w = models.random_dag(n, seed=0, cost_max=200 if n <= 1300000 else 60)
    v = LogView(w)
    spec = [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=0, thrash_kill=16, max_decisions=D)]
    b = P.DeviceBatch([w], spec, engine=P.ENGINE_GRID)
    s = torch.cuda.current_stream(dev)
    b.run(s)
    torch.cuda.synchronize()
    row = b.result_rows()[0]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        b.pool_argmin(stream=s)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        out = b.pool_argmin(stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    o = out.cpu().numpy()
    t = sum(ts) / len(ts)
    ach = float(o[3]) / t / 1e9
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(f"pool_argmin_{n}")
    except Exception:
        pass
    return {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
            "traffic": traffic, "peak_source": peak_src, "kernel": "pool_argmin_kernel (K3+K4, h_DTR)",
            "workload": f"config5s random locality DAG n={n}, B=0.98*peak_total, pool after {int(row['decisions'])} "
                        f"decisions", "pool": int(o[4]), "bytes_per_launch": int(o[3]),
            "us_per_launch": t * 1e6, "launches": reps, "l2": "flushed before every launch",
            "decisions_per_s_score_only": 1.0 / t}


if __name__ == "__main__":
    main()
