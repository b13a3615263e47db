"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from gen import pools as G, traces as TR, dnn
from paper_2311_00591_b200 import coop
dev = torch.device("cuda:0")
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "search"):
    for mode, n, P in ((G.MODE_BENCH, 4096, 8), (G.MODE_SMALL, 32, 64), (G.MODE_BENCH, 1000, 8)):
        ss, c, s, r = G.bench_pools_host(mode, 3, 0, P, n)
        d = [torch.from_numpy(ss.view(np.int64)).to(dev), torch.from_numpy(c).to(dev),
             torch.from_numpy(s).to(dev), torch.from_numpy(r.view(np.int64)).to(dev)]
        out = torch.empty(P * 4, dtype=torch.int64, device=dev)
        coop.window_search_batched(*d, out, P, n, n)
        torch.cuda.synchronize()
    # ties everywhere (every start a candidate): the re-walk rounds of the rare path
    n = 600
    ss = G.pack([8] * n, [G.EVICTABLE] * n)
    SS, C, S = G.stack_pools([(ss, np.full(n, 0.1), np.ones(n))] * 2)
    d = [torch.from_numpy(SS.view(np.int64)).to(dev), torch.from_numpy(C).to(dev),
         torch.from_numpy(S).to(dev), torch.from_numpy(np.array([80, 8 * 500], np.uint64).view(np.int64)).to(dev)]
    out = torch.empty(2 * 4, dtype=torch.int64, device=dev)
    coop.window_search_batched(*d, out, 2, n, n)
    torch.cuda.synchronize()
    print("search ok")
if which in ("all", "replay"):
    t = coop.Trace(TR.fig2_trace())
    t.replay([250 << 20, 200 << 20], 3)
    t.replay([250 << 20], coop.F_POLICY_DTR)
    t2 = coop.Trace(dnn.unet())
    pk = t2.peak_live(3)
    t2.replay([pk // 2], 3)
    t2.snapshots(pk // 2, 3, 1024, 64)
    print("replay ok")
if which in ("all", "pool"):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    import pool_model as PM
    calls = PM.random_session(5, 40, budget=300, flags=3)
    PM.drive(coop.Pool(300, 3), calls)
    print("pool ok")
