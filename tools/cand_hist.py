"""Candidate-count histogram of the search (variants/cnt.so writes 1000 + candidates into
n_evict for pools that reach verification, 500 when the exact best wins outright)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import collections
import numpy as np, torch
from gen import pools as G
from paper_2311_00591_b200 import coop
P, n = 65536, 4096
ss, c, s, r = G.bench_pools_host(G.MODE_BENCH, 0, 0, P, n)
d = [torch.from_numpy(ss.view(np.int64)).cuda(), torch.from_numpy(c).cuda(), torch.from_numpy(s).cuda(),
     torch.from_numpy(r.view(np.int64)).cuda()]
out = torch.empty(P * 4, dtype=torch.int64, device="cuda")
coop.window_search_batched(*d, out, P, n, n)
torch.cuda.synchronize()
w = coop.windows_from_device(out)
ne = w["n_evict"]
long_ = (np.arange(P) % 2 == 1) & (w["status"] == 0)
h = collections.Counter()
for v in ne[long_]:
    h[int(v) if v >= 500 else -1] += 1
print("long pools:", long_.sum(), sorted(h.items())[:30])
short = (np.arange(P) % 2 == 0) & (w["status"] == 0)
print("short pools with n_evict>=500:", int((ne[short] >= 500).sum()), "of", short.sum())
