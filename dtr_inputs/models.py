"""Seeded synthetic op-log generators shaped like the paper's workloads.

Input preparation only (no method arithmetic). Recipe:

* Each model is written as a forward program of tensor operators; a reverse-mode
  pass mirrors it (grad(x) = f'(saved inputs/outputs, grad(y)), P:1730-1736 for
  the linear case, generalised per operator kind); weight gradients dW = f(x, dy)
  are outputs kept to the end (ENSURE, reading C-11). Weights themselves are not
  tensors of the log (reading C-18: a constant memory offset).
* Costs are integers proportional to each operator's FLOPs (bytes for
  elementwise ops), >= 1, with optional +/-5% seeded jitter; scaled so
  base compute <= 2^27 (reading C-14). Memory is in KiB (>= 1).
* RELEASE records follow reference-count liveness: a tensor is released right
  after the last operator that reads it, unless it is an output.

Every generator returns the encoded log (np.ndarray[u32], see logfmt).
"""
from __future__ import annotations

import math

import numpy as np

from .logfmt import LogBuilder, LogView, assemble, OP_MAKE, OP_SHIFT, MAX_BASE

MODEL_IDS = {
    "linear": 1, "resnet32": 2, "densenet100": 3, "unet": 4, "lstm": 5,
    "treelstm": 6, "transformer": 7, "random_dag": 8, "random_small": 9,
}


# ---------------------------------------------------------------------------
# Config 1: the linear feed-forward network of App. A
# ---------------------------------------------------------------------------

def linear(N: int, *, ensure_output: bool = False) -> np.ndarray:
    """t_1 = f_1(); t_i = f_i(t_{i-1}); t^_N = f^_N(t_{N-1});
    t^_i = f^_i(t_{i-1}, t^_{i+1}); t^_1 = f^_1(t^_2). Unit mem and compute.
    Releases per P:1814-1816: t_N right after it is computed, t_{N-1} after t^_N,
    t_{i-1} and t^_{i+1} after t^_i. t^_1 is the only live tensor at the end."""
    b = LogBuilder(model_id=MODEL_IDS["linear"])
    t = [None] * (N + 1)
    g = [None] * (N + 2)
    t[1] = b.make(1, 1, [])
    for i in range(2, N + 1):
        t[i] = b.make(1, 1, [t[i - 1]])
    b.release(t[N])
    g[N] = b.make(1, 1, [t[N - 1]])
    b.release(t[N - 1])
    for i in range(N - 1, 1, -1):
        g[i] = b.make(1, 1, [t[i - 1], g[i + 1]])
        b.release(t[i - 1])
        b.release(g[i + 1])
    g[1] = b.make(1, 1, [g[2]])
    b.release(g[2])
    if ensure_output:
        b.ensure(g[1])
    return b.build()


# ---------------------------------------------------------------------------
# A tiny reverse-mode "tape" that writes a program of (mem, flops, parents)
# ---------------------------------------------------------------------------

class Tape:
    """Forward program + mirrored backward program, emitted as a simrd log."""

    def __init__(self, name: str, seed: int = 0, jitter: float = 0.05, elt_bytes: int = 4):
        self.name = name
        self.seed = seed
        self.jitter = jitter
        self.eb = elt_bytes
        self.nodes = []        # (bytes, flops, parents)
        self.fwd = []          # (kind, out, ins, info)
        self.requires = []     # per node: needs a gradient
        self.keep = []         # outputs kept to the end

    # -- forward ---------------------------------------------------------
    def _node(self, nbytes, flops, parents, requires=True):
        self.nodes.append((max(1, int(nbytes)), max(1.0, float(flops)), list(parents)))
        self.requires.append(requires)
        return len(self.nodes) - 1

    def size(self, x):
        return self.nodes[x][0]

    def input(self, numel):
        return self._node(numel * self.eb, numel, [], requires=False)

    def op(self, kind, ins, out_numel, flops, w_numel=0, **info):
        out = self._node(out_numel * self.eb, flops, ins,
                         requires=any(self.requires[i] for i in ins) or w_numel > 0)
        info["w_numel"] = w_numel
        info["flops"] = flops
        self.fwd.append((kind, out, list(ins), info))
        return out

    # convenience layers
    def conv(self, x, cin, cout, k, hout, wout, batch, stride=1):
        numel = batch * cout * hout * wout
        return self.op("wop", [x], numel, 2.0 * cin * cout * k * k * hout * wout * batch,
                       w_numel=cin * cout * k * k)

    def linear(self, x, batch, fin, fout):
        return self.op("wop", [x], batch * fout, 2.0 * batch * fin * fout, w_numel=fin * fout)

    def unary(self, kind, x, flops_per=1.0):
        n = self.size(x) // self.eb
        return self.op(kind, [x], n, flops_per * n)

    def bn(self, x):
        return self.unary("norm", x, 8.0)

    def relu(self, x):
        return self.unary("act_out", x, 1.0)

    def add(self, a, b):
        n = self.size(a) // self.eb
        return self.op("add", [a, b], n, n)

    def mul(self, a, b):
        n = self.size(a) // self.eb
        return self.op("mul", [a, b], n, n)

    def matmul(self, a, b, m, k, n, batch=1):
        return self.op("matmul", [a, b], batch * m * n, 2.0 * batch * m * k * n)

    def concat(self, xs):
        n = sum(self.size(x) for x in xs) // self.eb
        return self.op("concat", xs, n, n)

    def slice(self, x, numel):
        return self.op("slice", [x], numel, numel)

    def pool(self, x, out_numel, kind="avgpool"):
        return self.op(kind, [x], out_numel, self.size(x) // self.eb)

    def loss(self, x):
        out = self.op("loss", [x], 1, 4.0 * (self.size(x) // self.eb))
        return out

    # -- backward --------------------------------------------------------
    def backward(self, loss):
        """Reverse-mode pass mirroring the forward (P:1730-1736 generalised)."""
        grad = {}

        def acc(x, g):
            if not self.requires[x]:
                return
            if x in grad:
                n = self.size(x) // self.eb
                grad[x] = self._node(self.size(x), n, [grad[x], g])
            else:
                grad[x] = g

        for kind, out, ins, info in reversed(self.fwd):
            if kind == "loss":
                (x,) = ins
                acc(x, self._node(self.size(x), self.size(x) // self.eb * 4.0, [x]))
                continue
            if out not in grad:
                continue
            gy = grad[out]
            fl = info["flops"]
            if kind == "wop":
                (x,) = ins
                if self.requires[x]:
                    acc(x, self._node(self.size(x), fl, [gy]))
                gw = self._node(info["w_numel"] * self.eb, fl, [x, gy])
                self.keep.append(gw)
            elif kind == "norm":
                (x,) = ins
                acc(x, self._node(self.size(x), fl * 1.5, [x, gy]))
            elif kind == "act_out":        # relu / sigmoid / tanh: f'(y) * dy
                (x,) = ins
                acc(x, self._node(self.size(x), fl, [out, gy]))
            elif kind == "act_in":         # gelu: f'(x) * dy
                (x,) = ins
                acc(x, self._node(self.size(x), fl * 2, [x, gy]))
            elif kind == "softmax":
                (x,) = ins
                acc(x, self._node(self.size(x), fl, [out, gy]))
            elif kind == "add":
                for x in ins:
                    acc(x, gy)
            elif kind == "mul":
                a, b = ins
                if self.requires[a]:
                    acc(a, self._node(self.size(a), fl, [gy, b]))
                if self.requires[b]:
                    acc(b, self._node(self.size(b), fl, [gy, a]))
            elif kind == "matmul":
                a, b = ins
                if self.requires[a]:
                    acc(a, self._node(self.size(a), fl, [gy, b]))
                if self.requires[b]:
                    acc(b, self._node(self.size(b), fl, [a, gy]))
            elif kind == "concat":
                for x in ins:
                    if self.requires[x]:
                        acc(x, self._node(self.size(x), self.size(x) // self.eb, [gy]))
            elif kind == "slice":
                (x,) = ins
                acc(x, self._node(self.size(x), self.size(x) // self.eb, [gy]))
            elif kind in ("avgpool", "scale"):
                (x,) = ins
                acc(x, self._node(self.size(x), self.size(x) // self.eb, [gy]))
            elif kind == "maxpool":
                (x,) = ins
                acc(x, self._node(self.size(x), self.size(x) // self.eb, [x, out, gy]))
            else:
                raise ValueError(kind)
        self.keep.append(loss)
        return grad

    # -- emission ----------------------------------------------------------
    def emit(self, ensure_outputs: bool = True, target_base: int = 1 << 22) -> np.ndarray:
        rng = np.random.default_rng(self.seed)
        flops = np.array([f for (_, f, _) in self.nodes], dtype=np.float64)
        unit = max(flops.sum() / target_base, 1e-12)
        costs = np.maximum(1, np.rint(flops / unit)).astype(np.int64)
        if self.jitter > 0:
            j = 1.0 + rng.uniform(-self.jitter, self.jitter, size=len(costs))
            costs = np.maximum(1, np.rint(costs * j)).astype(np.int64)
        mems = [max(1, -(-nb // 1024)) for (nb, _, _) in self.nodes]
        last_use = [-1] * len(self.nodes)
        for j, (_, _, ps) in enumerate(self.nodes):
            for p in ps:
                last_use[p] = max(last_use[p], j)
        keep = set(self.keep)
        b = LogBuilder(model_id=MODEL_IDS.get(self.name, 0), seed=self.seed)
        for j, (_, _, ps) in enumerate(self.nodes):
            b.make(mems[j], int(costs[j]), ps)
            done = set()
            for p in ps:
                if p in done:
                    continue
                done.add(p)
                if last_use[p] == j and p not in keep:
                    b.release(p)
            if last_use[j] < 0 and j not in keep:
                b.release(j)
        if ensure_outputs:
            for k in sorted(keep):
                b.ensure(k)
        return b.build()


# ---------------------------------------------------------------------------
# Config 2/3/5 model shapes
# ---------------------------------------------------------------------------

def resnet32(batch: int = 128, seed: int = 0) -> np.ndarray:
    """CIFAR ResNet-32: stem + 3 stages x 5 basic blocks (conv-BN-ReLU-conv-BN-add-ReLU),
    1x1 conv shortcuts on downsampling, avgpool-fc-loss."""
    tp = Tape("resnet32", seed)
    x = tp.input(batch * 3 * 32 * 32)
    h = tp.relu(tp.bn(tp.conv(x, 3, 16, 3, 32, 32, batch)))
    c, s = 16, 32
    for stage, (cout, sout) in enumerate(((16, 32), (32, 16), (64, 8))):
        for blk in range(5):
            down = stage > 0 and blk == 0
            y = tp.relu(tp.bn(tp.conv(h, c, cout, 3, sout, sout, batch)))
            y = tp.bn(tp.conv(y, cout, cout, 3, sout, sout, batch))
            sc = tp.bn(tp.conv(h, c, cout, 1, sout, sout, batch)) if down else h
            h = tp.relu(tp.add(y, sc))
            c, s = cout, sout
    p = tp.pool(h, batch * c)
    logits = tp.linear(p, batch, c, 10)
    loss = tp.loss(logits)
    tp.backward(loss)
    return tp.emit()


def densenet100(batch: int = 64, k: int = 12, seed: int = 0) -> np.ndarray:
    """DenseNet-BC-100 (k=12): 3 dense blocks x 16 bottleneck layers; each layer
    concatenates ALL previous features of its block (fan-in up to 17)."""
    tp = Tape("densenet100", seed)
    x = tp.input(batch * 3 * 32 * 32)
    h = tp.conv(x, 3, 2 * k, 3, 32, 32, batch)
    c, s = 2 * k, 32
    for blk in range(3):
        feats = [h]
        for layer in range(16):
            cin = c + layer * k
            inp = feats[0] if len(feats) == 1 else tp.concat(feats)
            y = tp.conv(tp.relu(tp.bn(inp)), cin, 4 * k, 1, s, s, batch)
            y = tp.conv(tp.relu(tp.bn(y)), 4 * k, k, 3, s, s, batch)
            feats.append(y)
        c = c + 16 * k
        h = tp.concat(feats)
        if blk < 2:
            cout = c // 2
            h = tp.conv(tp.relu(tp.bn(h)), c, cout, 1, s, s, batch)
            s //= 2
            h = tp.pool(h, batch * cout * s * s)
            c = cout
    h = tp.relu(tp.bn(h))
    p = tp.pool(h, batch * c)
    logits = tp.linear(p, batch, c, 10)
    tp.backward(tp.loss(logits))
    return tp.emit()


def unet(batch: int = 4, base_ch: int = 32, size: int = 128, seed: int = 0) -> np.ndarray:
    """UNet: 4 down levels of 2x(conv-BN-ReLU)+maxpool, bottleneck, 4 up levels of
    upconv + concat(skip) + 2x(conv-BN-ReLU), 1x1 conv head + loss."""
    tp = Tape("unet", seed)
    x = tp.input(batch * 1 * size * size)
    h, c, s = x, 1, size
    skips = []

    def double(h, cin, cout, s):
        h = tp.relu(tp.bn(tp.conv(h, cin, cout, 3, s, s, batch)))
        return tp.relu(tp.bn(tp.conv(h, cout, cout, 3, s, s, batch)))

    ch = base_ch
    for lvl in range(4):
        h = double(h, c, ch, s)
        skips.append((h, ch, s))
        h = tp.pool(h, batch * ch * (s // 2) ** 2, kind="maxpool")
        c, s, ch = ch, s // 2, ch * 2
    h = double(h, c, ch, s)
    c = ch
    for lvl in reversed(range(4)):
        sk, skc, sks = skips[lvl]
        up = tp.conv(h, c, skc, 2, sks, sks, batch)      # transposed conv, same cost model
        h = tp.concat([sk, up])
        h = double(h, 2 * skc, skc, sks)
        c, s = skc, sks
    logits = tp.conv(h, c, 2, 1, s, s, batch)
    tp.backward(tp.loss(logits))
    return tp.emit()


def lstm(T: int = 256, layers: int = 2, hidden: int = 512, batch: int = 32,
         seed: int = 0) -> np.ndarray:
    """Multi-layer LSTM unrolled for T steps, ~12 single-output ops per cell:
    2 matmuls, add, 4 gate slices, 3 sigmoids + tanh, c = f*c + i*g, h = o*tanh(c)."""
    tp = Tape("lstm", seed)
    H = hidden
    hs = [None] * layers
    cs = [None] * layers
    outs = []
    for t in range(T):
        x = tp.input(batch * H)
        inp = x
        for l in range(layers):
            zx = tp.linear(inp, batch, H, 4 * H)
            if hs[l] is None:
                z = zx
            else:
                zh = tp.linear(hs[l], batch, H, 4 * H)
                z = tp.add(zx, zh)
            gi = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
            gf = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
            gg = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
            go = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
            ig = tp.mul(gi, gg)
            c = ig if cs[l] is None else tp.add(tp.mul(gf, cs[l]), ig)
            h = tp.mul(go, tp.unary("act_out", c, 4.0))
            hs[l], cs[l] = h, c
            inp = h
        outs.append(inp)
    logits = tp.linear(outs[-1], batch, H, 16)
    tp.backward(tp.loss(logits))
    return tp.emit(target_base=1 << 24)


def treelstm(depth: int = 8, hidden: int = 512, batch: int = 1, seed: int = 0) -> np.ndarray:
    """Child-sum TreeLSTM over a complete binary tree, ~15 ops per
    internal node; leaves embed an input."""
    tp = Tape("treelstm", seed)
    H = hidden

    def leaf():
        x = tp.input(batch * H)
        z = tp.linear(x, batch, H, 3 * H)
        i = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
        o = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
        u = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
        c = tp.mul(i, u)
        h = tp.mul(o, tp.unary("act_out", c, 4.0))
        return h, c

    def node(d):
        if d == 0:
            return leaf()
        hl, cl = node(d - 1)
        hr, cr = node(d - 1)
        hsum = tp.add(hl, hr)
        z = tp.linear(hsum, batch, H, 3 * H)
        i = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
        o = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
        u = tp.unary("act_out", tp.slice(z, batch * H), 4.0)
        fl = tp.unary("act_out", tp.linear(hl, batch, H, H), 4.0)
        fr = tp.unary("act_out", tp.linear(hr, batch, H, H), 4.0)
        c = tp.add(tp.mul(i, u), tp.add(tp.mul(fl, cl), tp.mul(fr, cr)))
        h = tp.mul(o, tp.unary("act_out", c, 4.0))
        return h, c

    h, _ = node(depth)
    logits = tp.linear(h, batch, H, 16)
    tp.backward(tp.loss(logits))
    return tp.emit(target_base=1 << 24)


def transformer(layers: int = 12, heads: int = 16, seq: int = 256, d_model: int = 512,
                batch: int = 8, seed: int = 0) -> np.ndarray:
    """Pre-LN Transformer encoder with per-head attention operators (seq 256):
    per head: slice q/k/v, scores = q k^T, softmax, attn = p v; per layer: LN, QKV,
    concat heads, out-proj, residual, LN, FFN (linear-GELU-linear), residual."""
    tp = Tape("transformer", seed)
    D, S, B, Hh = d_model, seq, batch, heads
    dh = D // Hh
    x = tp.input(B * S * D)
    h = x
    for _ in range(layers):
        a = tp.unary("norm", h, 8.0)
        q = tp.linear(a, B * S, D, D)
        k = tp.linear(a, B * S, D, D)
        v = tp.linear(a, B * S, D, D)
        outs = []
        for _h in range(Hh):
            qh = tp.slice(q, B * S * dh)
            kh = tp.slice(k, B * S * dh)
            vh = tp.slice(v, B * S * dh)
            sc = tp.matmul(qh, kh, S, dh, S, batch=B)
            p = tp.unary("softmax", sc, 5.0)
            outs.append(tp.matmul(p, vh, S, S, dh, batch=B))
        o = tp.linear(tp.concat(outs), B * S, D, D)
        h = tp.add(h, o)
        f = tp.unary("norm", h, 8.0)
        f = tp.unary("act_in", tp.linear(f, B * S, D, 4 * D), 8.0)
        f = tp.linear(f, B * S, 4 * D, D)
        h = tp.add(h, f)
    logits = tp.linear(tp.unary("norm", h, 8.0), B * S, D, 64)
    tp.backward(tp.loss(logits))
    return tp.emit(target_base=1 << 24)


# ---------------------------------------------------------------------------
# Stress / property-test graphs
# ---------------------------------------------------------------------------

def random_dag(n: int, seed: int = 0, window: int = 64, p_local: float = 0.9,
               mem_max: int = 1024, cost_max: int = 200) -> np.ndarray:
    """Config 5s: random locality DAG, 1-3 parents drawn from the previous `window`
    ids with probability p_local, otherwise uniformly; mem U[1,mem_max] KiB,
    cost U[1,cost_max]. Program = MAKE every tensor (no releases), so the whole
    graph stays referenced and the pool grows to ~n. Vectorised."""
    rng = np.random.default_rng(seed)
    k = rng.integers(1, 4, size=n)
    k[0] = 0
    k[1:] = np.minimum(k[1:], np.arange(1, n))
    par_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(k, out=par_off[1:])
    E = int(par_off[-1])
    child = np.repeat(np.arange(n, dtype=np.int64), k)
    local = rng.random(E) < p_local
    off = rng.integers(1, window + 1, size=E)
    loc = np.maximum(child - off, 0)
    uni = (rng.random(E) * np.maximum(child, 1)).astype(np.int64)
    par = np.where(local, loc, uni)
    par = np.minimum(par, child - 1)
    # dedup within each child's list (keep the first occurrence)
    order = np.lexsort((np.arange(E), par, child))
    cs, ps = child[order], par[order]
    dup = np.zeros(E, dtype=bool)
    dup[1:] = (cs[1:] == cs[:-1]) & (ps[1:] == ps[:-1])
    keep = np.ones(E, dtype=bool)
    keep[order[dup]] = False
    par = par[keep]
    child = child[keep]
    k = np.bincount(child, minlength=n)
    par_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(k, out=par_off[1:])
    mem = rng.integers(1, mem_max + 1, size=n)
    cost = rng.integers(1, cost_max + 1, size=n)
    ops = (np.uint64(OP_MAKE) << np.uint64(OP_SHIFT)) | np.arange(n, dtype=np.uint64)
    return assemble(mem, cost, par_off, par, ops.astype(np.uint32),
                    model_id=MODEL_IDS["random_dag"], seed=seed)


def hub_dag(n: int, seed: int = 0, n_hubs: int = 16, fan: int = 80, window: int = 64) -> np.ndarray:
    """random_dag plus hub tensors: ids 64..64+n_hubs-1 each become a parent of
    ~fan later tensors, so hubs have degree > 32 (the whole-GPU team's
    warp-cooperative neighbour walk).  MAKE only, like random_dag."""
    rng = np.random.default_rng(seed)
    base = random_dag(n, seed=seed, window=window)
    v = LogView(base)
    pars = [list(v.parents(t)) for t in range(n)]
    hubs = np.arange(64, 64 + n_hubs)
    p = n_hubs * fan / max(n - 64 - n_hubs, 1)
    for c in range(64 + n_hubs, n):
        if rng.random() < p:
            h = int(hubs[rng.integers(0, n_hubs)])
            if h not in pars[c]:
                pars[c].append(h)
    k = np.array([len(x) for x in pars])
    par_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(k, out=par_off[1:])
    par = np.array([q for x in pars for q in x], dtype=np.int64)
    ops = (np.uint64(OP_MAKE) << np.uint64(OP_SHIFT)) | np.arange(n, dtype=np.uint64)
    return assemble(v.mem.astype(np.int64), v.cost.astype(np.int64), par_off, par, ops.astype(np.uint32),
                    model_id=MODEL_IDS["random_dag"], seed=seed)


def random_program(n_make: int, seed: int = 0, max_parents: int = 3, window: int = 8,
                   mem_max: int = 4, cost_max: int = 4, p_release: float = 0.3,
                   p_get: float = 0.05, n_ensure: int = 2) -> np.ndarray:
    """Small random simrd programs for property tests: MAKE with 0..max_parents
    parents drawn from the `window` most recent referenced tensors, GET and
    RELEASE of referenced tensors, ENSURE of the last `n_ensure` live tensors.
    (REMAT's precondition m = bottom depends on replay state, so REMAT is
    exercised through the per-call API instead.)"""
    rng = np.random.default_rng(seed)
    b = LogBuilder(model_id=MODEL_IDS["random_small"], seed=seed)
    live = []
    for i in range(n_make):
        cand = live[-window:]
        kp = int(rng.integers(0, min(max_parents, len(cand)) + 1)) if cand else 0
        parents = [int(p) for p in rng.choice(cand, size=kp, replace=False)] if kp else []
        t = b.make(int(rng.integers(1, mem_max + 1)), int(rng.integers(1, cost_max + 1)), parents)
        live.append(t)
        if rng.random() < p_get and live:
            b.get(int(rng.choice(live)))
        if rng.random() < p_release and len(live) > 1:
            x = int(live[int(rng.integers(0, len(live) - 1))])
            b.release(x)
            if b.rho[x] == 0:
                live.remove(x)
    for t in live[-n_ensure:] if n_ensure else []:
        b.ensure(int(t))
    return b.build()


CONFIG_MODELS = {
    "resnet32": resnet32,
    "densenet100": densenet100,
    "unet": unet,
    "lstm": lstm,
    "treelstm": treelstm,
    "transformer": transformer,
}


def sweep_permilles(k: int = 30) -> list[int]:
    """permille = round(1000 * linspace(0.1, 1.0, k))."""
    return [int(round(1000 * x)) for x in np.linspace(0.1, 1.0, k)]
