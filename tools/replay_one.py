"""Time one replay cell on the GPU vs the oracle (for profiling)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import dnn
from paper_2311_00591_b200 import coop
from oracle import oracle as O
name = sys.argv[1]; frac = float(sys.argv[2]); ncell = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kw = {}
if name == "bilstm" and len(sys.argv) > 4: kw = {"seq_range": (int(sys.argv[4]), int(sys.argv[4]) + 2)}
tr = dnn.dnn(name, **kw)
h = coop.Trace(tr); peak = h.peak_live(3)
budgets = [int(peak * frac)] * ncell
out = torch.empty(ncell * 136, dtype=torch.uint8, device="cuda")
h.replay_device(budgets, 3, out); torch.cuda.synchronize()
t = time.time(); h.replay_device(budgets, 3, out); torch.cuda.synchronize(); dt = time.time() - t
r = out.cpu().numpy().view(coop.REPLAY_RESULT_DTYPE)[0]
t = time.time(); o, _ = O.replay(tr, budgets[0], 3); do = time.time() - t
print(name, frac, "gpu ms", round(dt * 1e3, 2), "oracle ms", round(do * 1e3, 2), "status", r["status"], o["status"],
      "press", r["pressure"], "remat", r["remat"], "evict", r["evictions"], "ops", tr.n_ops,
      "search_ns_total", r["search_ns_total"], "digest_eq", int(r["digest"]) == int(o["digest"]))
if os.environ.get("COOP_REPLAY_PHASES") == "1":
    import ctypes
    buf = np.zeros(8 * ncell, np.int64)
    coop.lib.coop__replay_phase_ns(ctypes.c_void_p(buf.ctypes.data), ncell)
    ev = max(1, buf[4])
    print("per event (us): view %.1f  closures %.1f  scans+ends %.1f  argmin+evict+splice %.1f  events %d" %
          tuple([buf[i] / ev / 1e3 for i in range(4)] + [buf[4]]))
