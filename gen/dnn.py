"""Synthetic allocation traces shaped like the paper's eight DNNs (input generation only).

The eight networks of the evaluation (R33):
GPT-3-style 2.7B, Swin-T, ResNet-50, Inception V3, U-Net, BiLSTM, SPOS, BERT Large.
Only their MEMORY SHAPE is modelled (tensor sizes, liveness, op order, cost densities):
each forward op records how its backward ops read saved tensors; `Net.backward()` emits
the mirrored backward with gradient accumulation; `Net.update()` emits the optimizer
step as in-place ops on the unevictable parameters / optimizer states.
Costs are Table 1 cost densities (us/MB, MB = MiB) times output MiB;
conv/matmul backward ops each cost the forward op's cost (2x in total).
Batch sizes and precisions are proposals (the paper's are only in Fig. 4's image,
PAPER.md:272); see DESIGN.md "Input recipe".
"""
from __future__ import annotations

import math

import numpy as np

from .traces import BWD, FWD, UPD, Builder, Trace

# Table 1 columns: (C1 conv/matmul, C2 norm, C2 activation) in us/MB
DENS = {"resnet50": (35.6, 5.0, 3.9), "gpt2": (33.5, 4.2, 3.8), "unet": (89.3, 5.3, 3.9),
        "swin": (32.7, 4.1, 3.9)}
MiB = 1 << 20


def _us(density: float, nbytes: int) -> int:
    return max(1, int(round(density * nbytes / MiB)))


class Net:
    """Forward-op recorder with a mirrored backward and an optimizer step."""

    def __init__(self, name: str, dens, optimizer: str = "sgd", dtype_bytes: int = 4):
        self.b = Builder(name)
        self.c1, self.cn, self.ca = dens
        self.opt = optimizer
        self.dt = dtype_bytes
        self.params = []        # current version of every parameter tensor
        self.opt_state = {}     # param index -> list of optimizer-state tensors
        self.tape = []          # forward records: (backward closure)
        self.pgrad = {}         # param index -> list of gradient tensors (accumulated)

    # ---------------------------------------------------------------- tensors
    def param(self, nbytes: int, n_states: int = None) -> int:
        """A parameter (unevictable) plus its optimizer states."""
        pid = len(self.params)
        self.params.append(self.b.param(nbytes))
        if n_states is None:
            n_states = {"sgd": 1, "adam": 2, "zero2": 3}[self.opt]
        sb = nbytes if self.opt != "zero2" else nbytes // 2  # ZeRO-2: fp32 shard = n/4*4 B
        self.opt_state[pid] = [self.b.param(max(1, sb)) for _ in range(n_states)]
        return pid

    def P(self, pid: int) -> int:
        return self.params[pid]

    def _op(self, ins, nbytes, cost, phase=FWD, inplace=-1):
        return self.b.op(ins, nbytes, cost, phase, inplace)

    def size(self, t: int) -> int:
        return self.b.size[t]

    # ---------------------------------------------------------------- forward ops
    def source(self, nbytes: int) -> int:
        """input batch / labels: a load op with no inputs (activation density)."""
        return self._op([], nbytes, _us(self.ca, nbytes))

    def linear(self, x: int, pid: int, out_bytes: int) -> int:
        """conv / matmul (C1): y = f(x, W)."""
        w = self.P(pid)
        cost = _us(self.c1, out_bytes)
        y = self._op([x, w], out_bytes, cost)

        def bwd(gy, G, w=w, x=x, pid=pid, cost=cost):
            gx = self._op([gy, w], self.size(x), cost, BWD)
            gw = self._op([gy, x], self.size(w), cost, BWD)
            self.pgrad.setdefault(pid, []).append(gw)
            G.add(x, gx)
        self.tape.append((y, bwd))
        return y

    def bmm(self, a: int, b: int, out_bytes: int) -> int:
        """activation x activation matmul (attention scores / context), C1."""
        cost = _us(self.c1, out_bytes)
        y = self._op([a, b] if a != b else [a], out_bytes, cost)

        def bwd(gy, G, a=a, b=b, cost=cost):
            ga = self._op([gy, b] if b != gy else [gy], self.size(a), cost, BWD)
            G.add(a, ga)
            if b != a:
                gb = self._op([gy, a], self.size(b), cost, BWD)
                G.add(b, gb)
        self.tape.append((y, bwd))
        return y

    def norm(self, x: int, pid: int) -> int:
        """batch / layer norm (C2)."""
        w = self.P(pid)
        y = self._op([x, w], self.size(x), _us(self.cn, self.size(x)))

        def bwd(gy, G, x=x, w=w, pid=pid):
            gx = self._op([gy, x, w], self.size(x), _us(self.cn, self.size(x)), BWD)
            gw = self._op([gy, x], self.size(w), _us(self.cn, self.size(x)), BWD)
            self.pgrad.setdefault(pid, []).append(gw)
            G.add(x, gx)
        self.tape.append((y, bwd))
        return y

    def act(self, x: int, inplace: bool = False) -> int:
        """ReLU / GELU / softmax / dropout (C2); inplace = relu_ (Sec. 3.5)."""
        n = self.size(x)
        y = self._op([x], n, _us(self.ca, n), inplace=x if inplace else -1)

        def bwd(gy, G, x=x, y=y, n=n):
            gx = self._op([gy, y], n, _us(self.ca, n), BWD)
            G.add(x, gx)
        self.tape.append((y, bwd))
        return y

    def add(self, a: int, b: int) -> int:
        n = self.size(a)
        y = self._op([a, b], n, _us(self.ca, n))

        def bwd(gy, G, a=a, b=b):
            G.add(a, gy)
            G.add(b, gy)
        self.tape.append((y, bwd))
        return y

    def reshape(self, xs, out_bytes: int) -> int:
        """pooling / concat / shuffle / patch-merge style data movement (C2)."""
        xs = list(xs)
        y = self._op(xs, out_bytes, _us(self.ca, out_bytes))

        def bwd(gy, G, xs=xs):
            for x in xs:
                gx = self._op([gy], self.size(x), _us(self.ca, self.size(x)), BWD)
                G.add(x, gx)
        self.tape.append((y, bwd))
        return y

    def ew(self, xs, out_bytes: int) -> int:
        """element-wise op on several inputs whose backward reads all of them (e.g. the
        LSTM cell updates c_t = f(gates_t, c_{t-1}), h_t = g(gates_t, c_t)), C2."""
        xs = list(xs)
        y = self._op(xs, out_bytes, _us(self.ca, out_bytes))

        def bwd(gy, G, xs=xs):
            for x in xs:
                gx = self._op([gy] + xs, self.size(x), _us(self.ca, self.size(x)), BWD)
                G.add(x, gx)
        self.tape.append((y, bwd))
        return y

    def loss(self, xs) -> int:
        xs = list(xs)
        tot = sum(self.size(x) for x in xs)
        y = self._op(xs, 4096, _us(self.ca, tot))

        def bwd(gy, G, xs=xs):
            for x in xs:
                gx = self._op([gy, x], self.size(x), _us(self.ca, self.size(x)), BWD)
                G.add(x, gx)
        self.tape.append((y, bwd))
        return y

    # ---------------------------------------------------------------- backward / update
    class _Grads:
        def __init__(self, net):
            self.net = net
            self.g = {}

        def add(self, t, g):
            if t in self.g:  # gradient accumulation (C2)
                n = self.net.size(t)
                self.g[t] = self.net._op([self.g[t], g], n, _us(self.net.ca, n), BWD)
            else:
                self.g[t] = g

    def backward(self, loss_t: int) -> None:
        G = Net._Grads(self)
        G.g[loss_t] = self._op([loss_t], 4096, 1, BWD)
        for y, bwd in reversed(self.tape):
            if y in G.g:
                bwd(G.g.pop(y), G)
        self.tape = []

    def update(self) -> None:
        """Optimizer step: in-place updates of parameters and optimizer states."""
        for pid in sorted(self.pgrad):
            gs = self.pgrad[pid]
            g = gs[0]
            for h in gs[1:]:
                g = self._op([g, h], self.size(g), _us(self.ca, self.size(g)), UPD)
            w = self.params[pid]
            st = self.opt_state[pid]
            nw = self.size(w)
            if self.opt == "sgd":  # momentum SGD: m <- mu m + g ; w <- w - lr m
                m = self._op([st[0], g], self.size(st[0]), _us(self.ca, nw), UPD, inplace=st[0])
                st[0] = m
                self.params[pid] = self._op([w, m], nw, _us(self.ca, nw), UPD, inplace=w)
            elif self.opt == "adam":
                m = self._op([st[0], g], self.size(st[0]), _us(self.ca, nw), UPD, inplace=st[0])
                v = self._op([st[1], g], self.size(st[1]), _us(self.ca, nw), UPD, inplace=st[1])
                st[0], st[1] = m, v
                self.params[pid] = self._op([w, m, v], nw, _us(self.ca, nw), UPD, inplace=w)
            else:  # ZeRO-2: reduce-scatter, shard Adam, all-gather in place
                gs_ = self._op([g], self.size(st[0]), _us(self.ca, nw), UPD)
                m = self._op([st[1], gs_], self.size(st[1]), _us(self.ca, self.size(st[1])), UPD, inplace=st[1])
                v = self._op([st[2], gs_], self.size(st[2]), _us(self.ca, self.size(st[2])), UPD, inplace=st[2])
                ms = self._op([st[0], m, v], self.size(st[0]), _us(self.ca, self.size(st[0])), UPD, inplace=st[0])
                st[0], st[1], st[2] = ms, m, v
                self.params[pid] = self._op([w, ms], nw, _us(self.ca, nw), UPD, inplace=w)
        self.pgrad = {}

    def build(self) -> Trace:
        return self.b.build()


# =============================================================================== models
def _conv_bn_relu(net, x, cin, cout, k, H, B, stride=1, relu=True, inplace=True):
    Ho = H // stride
    w = net.param(k * k * cin * cout * 4)
    y = net.linear(x, w, B * cout * Ho * Ho * 4)
    y = net.norm(y, net.param(2 * cout * 4))
    if relu:
        y = net.act(y, inplace=inplace)
    return y, Ho


def resnet50(B=64, iters=2) -> Trace:
    net = Net("resnet50", DENS["resnet50"], "sgd")
    for _ in range(iters):
        x = net.source(B * 3 * 224 * 224 * 4)
        y, H = _conv_bn_relu(net, x, 3, 64, 7, 224, B, 2)
        y = net.reshape([y], B * 64 * 56 * 56 * 4)  # maxpool
        H, cin = 56, 64
        for mid, out, n_blocks, stride in ((64, 256, 3, 1), (128, 512, 4, 2), (256, 1024, 6, 2),
                                           (512, 2048, 3, 2)):
            for bi in range(n_blocks):
                s = stride if bi == 0 else 1
                z, _ = _conv_bn_relu(net, y, cin, mid, 1, H, B)
                z, Ho = _conv_bn_relu(net, z, mid, mid, 3, H, B, s)
                z, _ = _conv_bn_relu(net, z, mid, out, 1, Ho, B, relu=False)
                sc = y
                if bi == 0:
                    sc, _ = _conv_bn_relu(net, y, cin, out, 1, H, B, s, relu=False)
                y = net.add(z, sc)
                y = net.act(y, inplace=True)
                H, cin = Ho, out
        y = net.reshape([y], B * 2048 * 4)  # global average pool
        y = net.linear(y, net.param(2048 * 1000 * 4), B * 1000 * 4)
        l = net.loss([y])
        net.backward(l)
        net.update()
    return net.build()


def inception_v3(B=64, iters=2) -> Trace:
    net = Net("inception_v3", DENS["resnet50"], "sgd")

    def cbr(x, cin, cout, k, H, stride=1):
        return _conv_bn_relu(net, x, cin, cout, k, H, B, stride)[0]

    def act_bytes(c, H):
        return B * c * H * H * 4

    for _ in range(iters):
        x = net.source(act_bytes(3, 299))
        y = cbr(x, 3, 32, 3, 298, 2)       # 149
        y = cbr(y, 32, 32, 3, 147)
        y = cbr(y, 32, 64, 3, 147)
        y = net.reshape([y], act_bytes(64, 73))
        y = cbr(y, 64, 80, 1, 73)
        y = cbr(y, 80, 192, 3, 71)
        y = net.reshape([y], act_bytes(192, 35))
        cin, H = 192, 35
        for pf in (32, 64, 64):            # Inception A x3
            b1 = cbr(y, cin, 64, 1, H)
            b2 = cbr(cbr(y, cin, 48, 1, H), 48, 64, 5, H)
            b3 = cbr(cbr(cbr(y, cin, 64, 1, H), 64, 96, 3, H), 96, 96, 3, H)
            b4 = cbr(net.reshape([y], act_bytes(cin, H)), cin, pf, 1, H)
            cin = 64 + 64 + 96 + pf
            y = net.reshape([b1, b2, b3, b4], act_bytes(cin, H))
        b1 = cbr(y, cin, 384, 3, H, 2)     # Inception B (reduction to 17)
        b2 = cbr(cbr(cbr(y, cin, 64, 1, H), 64, 96, 3, H), 96, 96, 3, H, 2)
        b3 = net.reshape([y], act_bytes(cin, 17))
        cin, H = 384 + 96 + cin, 17
        y = net.reshape([b1, b2, b3], act_bytes(cin, H))
        for c7 in (128, 160, 160, 192):    # Inception C x4
            b1 = cbr(y, cin, 192, 1, H)
            b2 = cbr(cbr(cbr(y, cin, c7, 1, H), c7, c7, 3, H), c7, 192, 3, H)
            t = cbr(y, cin, c7, 1, H)
            for _k in range(3):
                t = cbr(t, c7, c7, 3, H)
            b3 = cbr(t, c7, 192, 3, H)
            b4 = cbr(net.reshape([y], act_bytes(cin, H)), cin, 192, 1, H)
            cin = 768
            y = net.reshape([b1, b2, b3, b4], act_bytes(cin, H))
        b1 = cbr(cbr(y, cin, 192, 1, H), 192, 320, 3, H, 2)   # Inception D (to 8)
        t = cbr(y, cin, 192, 1, H)
        t = cbr(cbr(t, 192, 192, 3, H), 192, 192, 3, H)
        b2 = cbr(t, 192, 192, 3, H, 2)
        b3 = net.reshape([y], act_bytes(cin, 8))
        cin, H = 320 + 192 + cin, 8
        y = net.reshape([b1, b2, b3], act_bytes(cin, H))
        for _e in range(2):                # Inception E x2
            b1 = cbr(y, cin, 320, 1, H)
            t = cbr(y, cin, 384, 1, H)
            b2 = net.reshape([cbr(t, 384, 384, 3, H), cbr(t, 384, 384, 3, H)], act_bytes(768, H))
            t = cbr(cbr(y, cin, 448, 1, H), 448, 384, 3, H)
            b3 = net.reshape([cbr(t, 384, 384, 3, H), cbr(t, 384, 384, 3, H)], act_bytes(768, H))
            b4 = cbr(net.reshape([y], act_bytes(cin, H)), cin, 192, 1, H)
            cin = 320 + 768 + 768 + 192
            y = net.reshape([b1, b2, b3, b4], act_bytes(cin, H))
        y = net.reshape([y], B * cin * 4)
        y = net.linear(y, net.param(cin * 1000 * 4), B * 1000 * 4)
        net.backward(net.loss([y]))
        net.update()
    return net.build()


def swin_t(B=64, iters=2) -> Trace:
    net = Net("swin_t", DENS["swin"], "sgd")
    for _ in range(iters):
        x = net.source(B * 3 * 224 * 224 * 4)
        C, H = 96, 56
        y = net.linear(x, net.param(4 * 4 * 3 * C * 4), B * C * H * H * 4)  # patch embed
        y = net.norm(y, net.param(2 * C * 4))
        for si, (depth, heads) in enumerate(((2, 3), (2, 6), (6, 12), (2, 24))):
            if si > 0:  # patch merging: 2x2 neighbourhood concat + LN + linear 4C -> 2C
                m = net.reshape([y], B * 4 * C * (H // 2) ** 2 * 4)
                m = net.norm(m, net.param(2 * 4 * C * 4))
                H, C = H // 2, C * 2
                y = net.linear(m, net.param(4 * (C // 2) * C * 4), B * C * H * H * 4)
            tok = B * H * H
            for _d in range(depth):
                z = net.norm(y, net.param(2 * C * 4))
                qkv = net.linear(z, net.param(C * 3 * C * 4), tok * 3 * C * 4)
                scores = net.bmm(qkv, qkv, tok * heads * 49 * 4)   # 7x7 windows
                p = net.act(scores)                                 # softmax
                ctx = net.bmm(p, qkv, tok * C * 4)
                o = net.linear(ctx, net.param(C * C * 4), tok * C * 4)
                y = net.add(y, o)
                z = net.norm(y, net.param(2 * C * 4))
                h = net.linear(z, net.param(C * 4 * C * 4), tok * 4 * C * 4)
                h = net.act(h)                                      # GELU
                h = net.linear(h, net.param(4 * C * C * 4), tok * C * 4)
                y = net.add(y, h)
        y = net.norm(y, net.param(2 * C * 4))
        y = net.reshape([y], B * C * 4)
        y = net.linear(y, net.param(C * 1000 * 4), B * 1000 * 4)
        net.backward(net.loss([y]))
        net.update()
    return net.build()


def unet(B=8, iters=2, base=64, size=256) -> Trace:
    net = Net("unet", DENS["unet"], "sgd")

    def dconv(x, cin, cout, H):
        y, _ = _conv_bn_relu(net, x, cin, cout, 3, H, B)
        y, _ = _conv_bn_relu(net, y, cout, cout, 3, H, B)
        return y

    for _ in range(iters):
        x = net.source(B * 3 * size * size * 4)
        skips, cin, H = [], 3, size
        for lvl in range(4):
            c = base << lvl
            x = dconv(x, cin, c, H)
            skips.append((x, c, H))
            x = net.reshape([x], B * c * (H // 2) ** 2 * 4)  # maxpool
            cin, H = c, H // 2
        x = dconv(x, cin, base << 4, H)
        cin = base << 4
        for s, c, Hs in reversed(skips):
            up = net.linear(x, net.param(2 * 2 * cin * c * 4), B * c * Hs * Hs * 4)  # up-conv
            x = net.reshape([up, s], B * 2 * c * Hs * Hs * 4)                      # concat skip
            x = dconv(x, 2 * c, c, Hs)
            cin, H = c, Hs
        y = net.linear(x, net.param(cin * 2 * 4), B * 2 * H * H * 4)
        net.backward(net.loss([y]))
        net.update()
    return net.build()


def bilstm(B=64, iters=2, hidden=1024, layers=2, seed=0, seq_range=(16, 40)) -> Trace:
    """2-layer bidirectional LSTM; the sequence length is redrawn every iteration (a
    dynamic network)."""
    net = Net("bilstm", DENS["gpt2"], "sgd")
    rng = np.random.default_rng(seed)
    Hb = B * hidden * 4
    Ws = {}
    for l in range(layers):
        din = hidden if l == 0 else 2 * hidden
        for d in (0, 1):
            Ws[(l, d)] = net.param((din + hidden) * 4 * hidden * 4)
    for _ in range(iters):
        T = int(rng.integers(seq_range[0], seq_range[1] + 1))
        xs = [net.source(Hb) for _ in range(T)]
        for l in range(layers):
            outs = {}
            for d in (0, 1):
                h = c = None
                order = range(T) if d == 0 else range(T - 1, -1, -1)
                for t in order:
                    ins = [xs[t]] + ([h] if h is not None else [])
                    g = net.linear(ins[0] if h is None else net.reshape(ins, 2 * Hb), Ws[(l, d)], 4 * Hb)
                    gate = net.act(g)  # sigmoid / tanh of the four gates
                    c = net.ew([gate] + ([c] if c is not None else []), Hb)  # c_t
                    h = net.ew([gate, c], Hb)                               # h_t
                    outs[(d, t)] = h
            xs = [net.reshape([outs[(0, t)], outs[(1, t)]], 2 * Hb) for t in range(T)]
        net.backward(net.loss(xs))
        net.update()
    return net.build()


def spos(B=128, iters=2, seed=0) -> Trace:
    """ShuffleNetV2 single-path one-shot supernet: 20 choice blocks x 4 choices, a random
    path per iteration (a dynamic network)."""
    net = Net("spos", DENS["resnet50"], "sgd")
    rng = np.random.default_rng(seed)
    chans = [(64, 4, 56), (160, 4, 28), (320, 8, 14), (640, 4, 7)]
    # supernet parameters: every choice of every block exists (shared across iterations)
    for _ in range(iters):
        x = net.source(B * 3 * 224 * 224 * 4)
        y, _ = _conv_bn_relu(net, x, 3, 16, 3, 224, B, 2)
        y = net.reshape([y], B * 16 * 56 * 56 * 4)
        cin, H = 16, 56
        for cout, n, Hs in chans:
            for bi in range(n):
                k = int(rng.choice([3, 5, 7, 9]))  # 9 = xception-style stack
                stride = 2 if (bi == 0 and Hs != H) else 1
                Ho = H // stride
                half = cout // 2
                mid_in = cin if stride == 2 else cin // 2
                z, _ = _conv_bn_relu(net, y, mid_in, half, 1, H, B)
                reps = 3 if k == 9 else 1
                for _r in range(reps):
                    kk = 3 if k == 9 else k
                    z = net.linear(z, net.param(kk * kk * half * 4), B * half * Ho * Ho * 4)  # dw
                    z = net.norm(z, net.param(2 * half * 4))
                    z, _ = _conv_bn_relu(net, z, half, half, 1, Ho, B)
                if stride == 2:
                    p = net.linear(y, net.param(3 * 3 * cin * 4), B * cin * Ho * Ho * 4)
                    p = net.norm(p, net.param(2 * cin * 4))
                    p, _ = _conv_bn_relu(net, p, cin, half, 1, Ho, B)
                else:
                    p = net.reshape([y], B * half * Ho * Ho * 4)  # channel split
                y = net.reshape([p, z], B * cout * Ho * Ho * 4)   # concat + shuffle
                cin, H = cout, Ho
        y, _ = _conv_bn_relu(net, y, cin, 1024, 1, H, B)
        y = net.reshape([y], B * 1024 * 4)
        y = net.linear(y, net.param(1024 * 1000 * 4), B * 1000 * 4)
        net.backward(net.loss([y]))
        net.update()
    return net.build()


def _transformer(name, layers, d, heads, seq, B, vocab, optimizer, dt, dens, iters, lm_head):
    net = Net(name, dens, optimizer, dt)
    tok = B * seq
    wte = net.param(vocab * d * dt)
    wpe = net.param(seq * d * dt)
    L = []
    for _ in range(layers):
        L.append(dict(ln1=net.param(2 * d * dt), qkv=net.param((3 * d * d + 3 * d) * dt),
                      proj=net.param((d * d + d) * dt), ln2=net.param(2 * d * dt),
                      fc1=net.param((4 * d * d + 4 * d) * dt), fc2=net.param((4 * d * d + d) * dt)))
    lnf = net.param(2 * d * dt)
    for _ in range(iters):
        ids = net.source(tok * 8)
        x = net.linear(ids, wte, tok * d * dt)            # embedding lookup
        x = net.add(x, net.linear(ids, wpe, tok * d * dt))
        for p in L:
            z = net.norm(x, p["ln1"])
            qkv = net.linear(z, p["qkv"], tok * 3 * d * dt)
            s = net.bmm(qkv, qkv, B * heads * seq * seq * dt)
            s = net.act(s)                                  # softmax
            s = net.act(s)                                  # dropout
            ctx = net.bmm(s, qkv, tok * d * dt)
            o = net.act(net.linear(ctx, p["proj"], tok * d * dt))   # proj + dropout
            x = net.add(x, o)
            z = net.norm(x, p["ln2"])
            h = net.act(net.linear(z, p["fc1"], tok * 4 * d * dt))  # fc1 + GELU
            h = net.act(net.linear(h, p["fc2"], tok * d * dt))      # fc2 + dropout
            x = net.add(x, h)
        x = net.norm(x, lnf)
        if lm_head:
            x = net.linear(x, wte, tok * vocab * dt)        # tied LM head
        net.backward(net.loss([x]))
        net.update()
    return net.build()


def bert_large(B=16, iters=2) -> Trace:
    return _transformer("bert_large", 24, 1024, 16, 512, B, 30522, "adam", 4, DENS["gpt2"],
                        iters, lm_head=False)


def gpt3_2p7b(B=1, iters=2, layers=32) -> Trace:
    """GPT-3-style 2.7B (32 x d2560, 32 heads, seq 2048, fp16) trained with Adam under
    ZeRO-2 over 4 GPUs: fp16 parameters plus fp32 master/m/v shards."""
    return _transformer("gpt3_2.7b", layers, 2560, 32, 2048, B, 50257, "zero2", 2, DENS["gpt2"],
                        iters, lm_head=True)


DNNS = {"resnet50": resnet50, "inception_v3": inception_v3, "swin_t": swin_t, "unet": unet,
        "bilstm": bilstm, "spos": spos, "bert_large": bert_large, "gpt3_2.7b": gpt3_2p7b}


def dnn(name: str, **kw) -> Trace:
    return DNNS[name](**kw)
