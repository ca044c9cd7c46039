"""Phase profile (clock64 build) of the slowest config-2 cells."""
import ctypes as C, os, sys
os.environ["DTR_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "paper_2006_09616_b200", "libdtr_prof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2006_09616_b200 as P
import bench
P.lib.dtr_debug_profile.argtypes = [C.c_void_p, C.c_int]
logs, specs = bench.workload(0)
for s in specs:
    if not ((s["heuristic"] in (0, 1) and s["budget"] < 60000) or (s["heuristic"] == 3 and s["budget"] < 160000 and s["budget"] > 150000)):
        continue
    b = P.DeviceBatch(logs, [s], engine=P.ENGINE_CTA)
    b.run(); torch.cuda.synchronize()
    buf = np.zeros(16, np.uint64)
    P.lib.dtr_debug_profile(buf.ctypes.data, 1)
    b.run(); torch.cuda.synchronize()
    P.lib.dtr_debug_profile(buf.ctypes.data, 1)
    r = b.result_rows()[0]
    d = int(r["decisions"])
    print(f"h={s['heuristic']} B={s['budget']} dec={d} remats={int(r['remats'])} st={int(r['status'])} "
          f"resume={buf[0]/1e6:.2f}M cyc ({buf[0]/max(d,1):.0f}/dec) wscore={buf[1]/max(buf[3],1):.0f}/dec "
          f"wred={buf[2]/max(buf[3],1):.0f}/dec wdec={buf[3]} cta={buf[4]/max(buf[5],1):.0f}/dec ctadec={buf[5]} init={buf[6]}\n"
          f"    rec+evict {buf[8]/max(buf[9],1):.0f} x{buf[9]/max(d,1):.2f}/dec, complete_top {buf[10]/max(buf[11],1):.0f} x{buf[11]/max(d,1):.2f}/dec, "
          f"lock/push {buf[12]/max(buf[13],1):.0f} x{buf[13]/max(d,1):.2f}/dec, loop iters {buf[14]/max(d,1):.2f}/dec")
