"""The state-of-memory trace of PAPER.md App. A (Fig. "trace"):
DTR on the linear network with N = 200, B = 2 ceil(sqrt N), heuristic h_e*
 and V1 banishing (the setting Theorem 1 is proven in),
driven through the per-call runtime (dtr_compute / dtr_get / dtr_release on the
GPU) one log record at a time; after every record dtr_debug_state gives every
tensor's residency.  Row = record, column i = layer i: 0 = forward t_i and its
gradient not in memory, 1 = forward t_i resident, 1.5 = gradient t^_i resident.

  python tools/residency_trace.py [N] [OUT_PREFIX]   -> OUT.csv, OUT.pgm (image), summary on stdout
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2006_09616_b200 as P  # noqa: E402
from dtr_inputs import LogView, models  # noqa: E402
from dtr_inputs.logfmt import OP_GET, OP_MAKE, OP_RELEASE, OP_SHIFT  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    out = sys.argv[2] if len(sys.argv) > 2 else f"profiles/r02_residency_N{N}_estar_v1"
    B = 2 * math.ceil(math.sqrt(N))
    v = LogView(models.linear(N))
    rt = P.Runtime(P.HEURISTICS["estar"], budget=B, dealloc=P.DEALLOC["v1"], cap_tensors=4 * N, cap_edges=8 * N)
    rows = []
    for w in v.ops:
        op, t = int(w) >> OP_SHIFT, int(w) & ((1 << OP_SHIFT) - 1)
        if op == OP_MAKE:
            rc, got = rt.compute(int(v.mem[t]), int(v.cost[t]), v.parents(t))
            assert rc == 0 and got == t, (rc, got, t)
        elif op == OP_GET:
            assert rt.get(t) == 0
        elif op == OP_RELEASE:
            assert rt.release(t) == 0
        else:
            raise SystemExit(f"unexpected op {op}")
        st = rt.state()
        row = np.zeros(N, np.float32)
        for i in range(1, N + 1):               # forward t_i = id i - 1; gradient t^_i = id N + (N - i)
            f, g = i - 1, N + (N - i)
            if g < len(st) and st[g] == 1:
                row[i - 1] = 1.5
            elif f < len(st) and st[f] == 1:
                row[i - 1] = 1.0
        rows.append(row)
    s = rt.stats()
    img = np.array(rows)
    np.savetxt(out + ".csv", img, fmt="%.1f", delimiter=",")
    with open(out + ".pgm", "w") as f:          # plain PGM: 0 black, 1 grey, 1.5 white
        f.write(f"P2\n{img.shape[1]} {img.shape[0]}\n255\n")
        for r in img:
            f.write(" ".join(str(int(x / 1.5 * 255)) for x in r) + "\n")
    back = next(k for k, w in enumerate(v.ops) if int(w) >> OP_SHIFT == OP_MAKE and int(w) & ((1 << OP_SHIFT) - 1) == N)
    at_back = img[back]
    ckpt = [i + 1 for i in range(N) if at_back[i] == 1.0]
    print(f"N={N} B={B} h_e* V1: {int(s['computations'])} computations (C/2N = {int(s['computations']) / (2 * N):.3f}), "
          f"{int(s['decisions'])} decisions, {int(s['remats'])} remats, status {int(s['status'])}")
    print(f"resident forward tensors when the backward pass starts (record {back}): {ckpt}")
    print(f"wrote {out}.csv / {out}.pgm ({img.shape[0]} records x {N} layers)")


if __name__ == "__main__":
    main()
