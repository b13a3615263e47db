"""Latency of the online calls (coop_alloc / coop_access / coop_free) on one device pool:
a chain of allocations under pressure (every alloc after warm-up evicts a window)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_00591_b200 import coop
p = coop.Pool(1 << 20, coop.F_PARTITION | coop.F_INPLACE, max_tensors=8192, max_edges=16384)
rng = np.random.default_rng(0)
ids, lat_free, lat_press = [], [], []
for k in range(3000):
    size = int(rng.integers(1, 8192))
    par = [ids[-1]] if ids and p.access(ids[-1]) == coop.OK else []
    t = time.perf_counter()
    st, r, ev = p.alloc(size, int(rng.integers(1, 500)), coop.OP_PHASE_FWD, -1, par)
    dt = time.perf_counter() - t
    if st == coop.OK:
        ids.append(int(r["tensor_id"]))
        (lat_press if ev else lat_free).append(dt)
s = p.stats()
print(f"allocs {len(ids)}  no-eviction calls {len(lat_free)}: median {np.median(lat_free)*1e6:.1f} us; "
      f"eviction calls {len(lat_press)}: median {np.median(lat_press)*1e6:.1f} us, p99 "
      f"{np.percentile(lat_press, 99)*1e6:.1f} us; max blocks {s['max_blocks']}, evictions {s['evictions']}")
