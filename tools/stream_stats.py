"""Streaming search diagnostics: time the stream kernel alone (COOP_SEARCH_IMPL=stream_only)
and count the pools it leaves pending, on the bench workload."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import pools as G
from paper_2311_00591_b200 import coop
P = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
n = 4096
dev = torch.device("cuda:0")
ss = torch.empty(P * n, dtype=torch.int64, device=dev); c = torch.empty(P * n, dtype=torch.float64, device=dev)
s = torch.empty(P * n, dtype=torch.float64, device=dev); r = torch.empty(P, dtype=torch.int64, device=dev)
out = torch.empty(P * 4, dtype=torch.int64, device=dev)
G.bench_pools_device(G.MODE_BENCH, 0, 0, P, n, n, ss, c, s, r)
for _ in range(3):
    coop.window_search_batched(ss, c, s, r, out, P, n, n)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    coop.window_search_batched(ss, c, s, r, out, P, n, n)
e1.record(); torch.cuda.synchronize()
w = coop.windows_from_device(out)
st = w["status"]
print(os.environ.get("COOP_SEARCH_IMPL", "default"), "pools", P, "ms/launch", e0.elapsed_time(e1) / 5,
      "pending", int((st == 0x7fff0001).sum()), "status", {int(k): int(v) for k, v in zip(*np.unique(st, return_counts=True))})
