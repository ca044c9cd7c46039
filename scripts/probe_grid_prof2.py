"""Grid-engine phase profile on the config-4 LSTM (libdtr_prof.so): per-decision
leader / barrier / score / reduce cycles between decision D0 and D1."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["DTR_LIB"] = os.path.join(ROOT, "paper_2006_09616_b200", "libdtr_prof.so")
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
P.lib.dtr_debug_profile.argtypes = [C.c_void_p, C.c_int]
w = models.lstm(T=4096, layers=2); v = LogView(w)
B = v.peak_total * 100000 // v.n
for h in (0, 1):
    res = {}
    for D in (2000, 4000):
        b = P.DeviceBatch([w], [dict(log=0, budget=B, heuristic=h, max_decisions=D)], engine=P.ENGINE_GRID)
        buf = np.zeros(16, np.uint64)
        b.run(); torch.cuda.synchronize()
        P.lib.dtr_debug_profile(buf.ctypes.data, 1)
        b.run(); torch.cuda.synchronize()
        P.lib.dtr_debug_profile(buf.ctypes.data, 1)
        res[D] = (buf.astype(np.float64), b.result_rows()[0])
    d = res[4000][0] - res[2000][0]
    k = 2000
    r1, r0 = res[4000][1], res[2000][1]
    print(f"h={h} per decision (decisions 2000..4000): leader={d[0]/k:.0f} sync1={d[1]/k:.0f} score={d[2]/k:.0f} "
          f"blockred+partial={d[3]/k:.0f} sync2+final={d[4]/k:.0f} cycles; loop total={d[6]/k:.0f}; "
          f"evals/dec={(int(r1['cand_evals'])-int(r0['cand_evals']))/k:.0f} "
          f"bytes/dec={(int(r1['score_bytes'])-int(r0['score_bytes']))/k:.0f} "
          f"rec+evict={d[8]/max(d[9],1):.0f} complete_top={d[10]/max(d[11],1):.0f}x{d[11]/k:.2f} push={d[12]/max(d[13],1):.0f}x{d[13]/k:.2f}",
          flush=True)
