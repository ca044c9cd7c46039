"""Grid-engine phase profile (libdtr_prof.so)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["DTR_LIB"] = os.path.join(ROOT, "paper_2006_09616_b200", "libdtr_prof.so")
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
P.lib.dtr_debug_profile.argtypes = [C.c_void_p, C.c_int]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
w = models.random_dag(n, seed=0); v = LogView(w)
for h in (0, 1, 2):
    for D in (1, 201):
        b = P.DeviceBatch([w], [dict(log=0, budget=v.peak_total * 98 // 100, heuristic=h, max_decisions=D)],
                          engine=P.ENGINE_GRID)
        buf = np.zeros(8, np.uint64)
        b.run(); torch.cuda.synchronize()
        P.lib.dtr_debug_profile(buf.ctypes.data, 1)
        b.run(); torch.cuda.synchronize()
        P.lib.dtr_debug_profile(buf.ctypes.data, 1)
        r = b.result_rows()[0]
        k = max(int(buf[5]), 1)
        print(f"h={h} D={D} resume={buf[0]/1.965e3:.0f}us sync1={buf[1]/1.965e3:.0f}us score/dec={buf[2]/k:.0f}cyc "
              f"blockred/dec={buf[3]/k:.0f} sync2/dec={buf[4]/k:.0f} loop={buf[6]/1.965e3:.0f}us dec={k} "
              f"evals/dec={int(r['cand_evals'])/k:.0f} bytes/dec={int(r['score_bytes'])/k:.0f}", flush=True)
