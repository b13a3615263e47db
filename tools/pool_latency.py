"""Latency of the online calls (coop_alloc / coop_access / coop_free) on one device pool:
a chain of allocations under pressure (every alloc after warm-up evicts a window).
Measured twice: one launch per call (default) and the resident service (coop_pool_service)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_00591_b200 import coop


def session(idle_us):
    p = coop.Pool(1 << 20, coop.F_PARTITION | coop.F_INPLACE, max_tensors=8192, max_edges=16384,
                  service_idle_us=idle_us)
    rng = np.random.default_rng(0)
    ids, lat_free, lat_press, lat_acc = [], [], [], []
    transcript = []
    for k in range(3000):
        size = int(rng.integers(1, 8192))
        par = []
        if ids:
            t = time.perf_counter()
            a = p.access(ids[-1])
            lat_acc.append(time.perf_counter() - t)
            if a == coop.OK:
                par = [ids[-1]]
        t = time.perf_counter()
        st, r, ev = p.alloc(size, int(rng.integers(1, 500)), coop.OP_PHASE_FWD, -1, par)
        dt = time.perf_counter() - t
        transcript.append((st, int(r["addr"]), tuple(ev)))
        if st == coop.OK:
            ids.append(int(r["tensor_id"]))
            (lat_press if ev else lat_free).append(dt)
    s = p.stats()
    p.close()
    us = lambda x, q=50: np.percentile(x, q) * 1e6
    print(f"[{'service idle ' + str(idle_us) + ' us' if idle_us else 'launch per call'}] allocs {len(ids)}; "
          f"coop_access median {us(lat_acc):.1f} us; alloc without eviction ({len(lat_free)}): median "
          f"{us(lat_free):.1f} us; alloc with a window eviction ({len(lat_press)}): median {us(lat_press):.1f} us, "
          f"p99 {us(lat_press, 99):.1f} us; max blocks {s['max_blocks']}, evictions {s['evictions']}")
    return transcript


a = session(0)
b = session(100000)
print("identical transcripts:", a == b)
