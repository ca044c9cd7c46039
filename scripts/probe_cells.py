"""Per-cell CTA-engine time of the bench workload (config 2): which cell is the critical path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_09616_b200 as P
import bench
logs, specs = bench.workload(0)
names = {0: "dtr", 1: "dtr_eq", 2: "lru", 3: "size"}
res = []
for s in specs:
    b = P.DeviceBatch(logs, [s], engine=P.ENGINE_CTA)
    b.run(); b.run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
    r = b.result_rows()[0]
    ms = e0.elapsed_time(e1)
    res.append((ms, names[s["heuristic"]], s["budget"], int(r["decisions"]), int(r["remats"]), int(r["status"])))
b = P.DeviceBatch(logs, specs, engine=P.ENGINE_CTA)
b.run(); b.run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
print(f"LIB={os.environ.get('DTR_LIB', 'libdtr.so')} whole batch {e0.elapsed_time(e1):.3f} ms")
res.sort(reverse=True)
for ms, h, B, d, rm, st in res[:12]:
    print(f"{ms:8.3f} ms  {h:7s} B={B:9d} dec={d:6d} remats={rm:6d} st={st} us/dec={1000*ms/max(d,1):.2f}")
for name in names.values():                      # the slowest cells of each heuristic
    for ms, h, B, d, rm, st in [r for r in res if r[1] == name][:2]:
        print(f"  top {h:7s} {ms:8.3f} ms B={B:9d} dec={d:6d} remats={rm:6d} st={st} us/dec={1000*ms/max(d,1):.2f}")
tot = {}
for ms, h, B, d, rm, st in res:
    t = tot.setdefault(h, [0, 0]); t[0] += ms; t[1] += d
for h, (ms, d) in tot.items():
    print(f"{h:7s} sum {ms:8.2f} ms, {d} decisions, {1000*ms/d:.2f} us/dec")
