"""Per-phase clock64 deltas of thread 0 per pool (variants/clk.so writes 8 u32 deltas into
each 32-byte result): A+scan barrier, write-back, zero pass, merge, filter, candidates,
verification tail, end barrier."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import pools as G
from paper_2311_00591_b200 import coop
P, n = 148 * 64, 4096
ss, c, s, r = G.bench_pools_host(G.MODE_BENCH, 0, 0, P, n)
d = [torch.from_numpy(ss.view(np.int64)).cuda(), torch.from_numpy(c).cuda(), torch.from_numpy(s).cuda(),
     torch.from_numpy(r.view(np.int64)).cuda()]
out = torch.empty(P * 4, dtype=torch.int64, device="cuda")
for _ in range(2):
    coop.window_search_batched(*d, out, P, n, n)
torch.cuda.synchronize()
dl = out.cpu().numpy().view(np.uint32).reshape(P, 8).astype(np.float64)
names = ["A+scan", "writeback", "zero", "merge", "filter+red", "cand", "verify", "endbar"]
for label, m in (("short", np.arange(P) % 2 == 0), ("long", (np.arange(P) % 2 == 1) & (np.arange(P) % 64 != 63))):
    x = dl[m]
    print(label, {k: round(float(v)) for k, v in zip(names, x.mean(0))}, "total", round(float(x.sum(1).mean())))
