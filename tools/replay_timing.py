"""Time one replay sweep per DNN trace (256 budgets, 20-100 % of peak) on the GPU."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import dnn
from paper_2311_00591_b200 import coop
flags = 3
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for name in (sys.argv[2].split(",") if len(sys.argv) > 2 else dnn.DNNS):
    tr = dnn.dnn(name)
    h = coop.Trace(tr)
    peak = h.peak_live(flags)
    budgets = [peak * (20 * 255 + 80 * k) // (100 * 255) for k in range(256)][::256 // nb]
    out = torch.empty(len(budgets) * 136, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t = time.time()
    h.replay_device(budgets, flags, out)
    torch.cuda.synchronize()
    dt = time.time() - t
    r = out.cpu().numpy().view(coop.REPLAY_RESULT_DTYPE)
    print(f"{name:13s} cells {len(budgets)} ops {tr.n_ops} wall {dt*1e3:9.1f} ms  ok {(r['status']==0).sum()} "
          f"remat {r['remat'].sum()} evict {r['evictions'].sum()} press {r['pressure'].sum()} "
          f"ops/s {len(budgets)*tr.n_ops/dt:.3g}", flush=True)
    top = np.argsort(-r["search_ns_total"])[:4]
    print("   slowest cells (k, budget frac, search s, pressure, remat, status):",
          [(int(k * (256 // nb)), round(budgets[k] / peak, 3), round(r["search_ns_total"][k] / 1e9, 2),
            int(r["pressure"][k]), int(r["remat"][k]), int(r["status"][k])) for k in top], flush=True)
