"""Phase profile (clock64 build, libdtr_prof.so) of single config-5 cells:
python tools/probe_prof_c5.py MODEL HEUR PERMILLE [MAX_DECISIONS]"""
import ctypes as C, os, sys, time
os.environ["DTR_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2006_09616_b200", "libdtr_prof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
P.lib.dtr_debug_profile.argtypes = [C.c_void_p, C.c_int]
m, h, pm = sys.argv[1], sys.argv[2], int(sys.argv[3])
cap = int(sys.argv[4]) if len(sys.argv) > 4 else 0
w = models.CONFIG_MODELS[m]()
v = LogView(w)
s = dict(log=0, budget=v.budget(pm), heuristic=P.HEURISTICS[h], thrash_kill=16, max_decisions=cap)
b = P.DeviceBatch([w], [s], engine=P.ENGINE_CTA)
buf = np.zeros(32, np.uint64)
P.lib.dtr_debug_profile(buf.ctypes.data, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
P.lib.dtr_debug_profile(buf.ctypes.data, 1)
r = b.result_rows()[0]
d = int(r["decisions"])
ms = e0.elapsed_time(e1)
print(f"{m} {h} pm={pm} n={v.n} dec={d} remats={int(r['remats'])} st={int(r['status'])} {ms:.1f} ms "
      f"({ms * 1e3 / max(d, 1):.2f} us/dec) evals/dec={int(r['cand_evals']) / max(d, 1):.0f}\n"
      f"  resume={buf[0] / max(d, 1):.0f} cyc/dec  warp-team score={buf[1] / max(buf[3], 1):.0f} red={buf[2] / max(buf[3], 1):.0f} "
      f"x{buf[3]}  cta-team={buf[4] / max(buf[5], 1):.0f} x{buf[5]}  init={buf[6]}\n"
      f"  rec+evict {buf[8] / max(buf[9], 1):.0f} x{buf[9] / max(d, 1):.2f}/dec, complete_top {buf[10] / max(buf[11], 1):.0f} "
      f"x{buf[11] / max(d, 1):.2f}/dec, lock/push {buf[12] / max(buf[13], 1):.0f} x{buf[13] / max(d, 1):.2f}/dec, "
      f"loop iters {buf[14] / max(d, 1):.2f}/dec\n"
      f"  closure cache: hits {buf[16] / max(d, 1):.1f}/dec, lane walks {buf[17] / max(d, 1):.1f}/dec, "
      f"warp BFS {buf[18] / max(d, 1):.2f}/dec, events {buf[19] / max(d, 1):.2f}/dec, "
      f"event-walk nodes {buf[20] / max(d, 1):.1f}/dec, event cycles {buf[21] / max(d, 1):.0f}/dec\n"
      f"  stacked (slow/stale) {buf[22] / max(d, 1):.1f}/dec, resolved after pruning {buf[23] / max(d, 1):.1f}/dec, "
      f"multi-candidate walks {buf[24] / max(d, 1):.2f}/dec", flush=True)
