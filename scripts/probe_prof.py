"""Phase profile of the CTA engine (needs libdtr_prof.so: _build.py --profile)."""
import ctypes as C, os, sys
os.environ["DTR_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2006_09616_b200", "libdtr_prof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_09616_b200 as P
from dtr_inputs import models, LogView
P.lib.dtr_debug_profile.argtypes = [C.c_void_p, C.c_int]
clk = torch.cuda.get_device_properties(0).clock_rate if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1965000
w = models.resnet32(); v = LogView(w)
for h, pm in ((3, 400), (0, 400), (1, 400), (2, 400), (0, 1000)):
    b = P.DeviceBatch([w], [dict(log=0, budget=v.budget(pm), heuristic=h)], engine=P.ENGINE_CTA)
    b.run(); torch.cuda.synchronize()
    buf = np.zeros(8, np.uint64)
    P.lib.dtr_debug_profile(buf.ctypes.data, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.run(); e1.record(); torch.cuda.synchronize()
    P.lib.dtr_debug_profile(buf.ctypes.data, 1)
    r = b.result_rows()[0]
    d = int(r["decisions"]); rec = int(r["records_done"])
    print(f"h={h} pm={pm} ms={e0.elapsed_time(e1):.3f} dec={d} rec={rec} cyc: resume={buf[0]} ({buf[0]/max(d,1):.0f}/dec) "
          f"wscore={buf[1]} ({buf[1]/max(buf[3],1):.0f}/dec) wred={buf[2]} ({buf[2]/max(buf[3],1):.0f}/dec) wdec={buf[3]} "
          f"cta={buf[4]} ({buf[4]/max(buf[5],1):.0f}/dec) ctadec={buf[5]} init={buf[6]}")
