"""Full-coverage GPU parity (SURVEY.md 8(d) "Parity" column):

* config 5 -- EVERY one of the 2048 cells (8 DNN trace shapes x 256 budgets, 20-100 % of
  peak; Alg. 1) replayed by coop_replay_trace and by the O2 oracle (one
  process per host core): every integer counter, the status / failing op and the eviction
  digest (R29) bit-exact;
* config 4 -- 65,536 full-size pools (2^16 x 4096 blocks, the benchmark's own pools at the
  start and the end of its 2^20-pool range, in the launch configuration bench.py times)
  searched by coop_window_search_batched and by the O1 oracle: every field bit-exact.
"""
import numpy as np
import pytest

from gen import dnn
from gen import pools as G
from oracle import oracle as O
from oracle import parallel as OP

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2311_00591_b200 import coop  # noqa: E402

FIELDS = ["status", "fail_op", "base_us", "total_us", "evictions", "remat", "pressure",
          "frag_fail", "inplace_reuse", "heuristic_evals", "sum_free_bytes_after",
          "sum_free_blocks_after", "digest", "max_depth", "max_blocks", "budget", "n_events"]


def config5_cells(flags):
    cells = []
    for name in dnn.DNNS:
        peak = O.peak_live(dnn.dnn(name), flags)
        for k in range(256):
            cells.append((name, peak * (20 * 255 + 80 * k) // (100 * 255), k))
    return cells


def test_config5_every_cell_vs_oracle():
    flags = coop.F_PARTITION | coop.F_INPLACE
    cells = config5_cells(flags)
    want, wall, _, procs = OP.replay_cells(cells, flags)
    got = []
    for name in dnn.DNNS:
        t = coop.Trace(dnn.dnn(name))
        res, _ = t.replay([b for n2, b, _ in cells if n2 == name], flags)
        got.append(res)
        t.close()
    got = np.concatenate(got)
    assert len(got) == len(want) == 2048
    bad = []
    for i, (name, b, k) in enumerate(cells):
        g = {f: int(got[i][f]) for f in FIELDS}
        w = {f: int(want[i][f]) for f in FIELDS}
        if g != w:
            bad.append((name, k, g, w))
    assert not bad, f"{len(bad)} of 2048 cells differ; first: {bad[0]}"
    st = got["status"]
    # the sweep exercises completed, unsatisfiable and heavily thrashing cells
    assert (st == 0).sum() > 1000 and (st == coop.ERR_UNSATISFIABLE).sum() > 100
    assert got["remat"].max() > 10000


@pytest.mark.parametrize("p0", [0, (1 << 20) - (1 << 15)])
def test_config4_full_size_32k_pools_vs_oracle(p0):
    """2 x 32,768 = 65,536 pools of the benchmark workload (MODE_BENCH, seed 0, N = 4096),
    generated on the device exactly as bench.py does."""
    P, n = 1 << 15, 4096
    dev = torch.device("cuda:0")
    ss = torch.empty(P * n, dtype=torch.int64, device=dev)
    c = torch.empty(P * n, dtype=torch.float64, device=dev)
    s = torch.empty(P * n, dtype=torch.float64, device=dev)
    r = torch.empty(P, dtype=torch.int64, device=dev)
    out = torch.empty(P * 4, dtype=torch.int64, device=dev)
    G.bench_pools_device(G.MODE_BENCH, 0, p0, P, n, n, ss, c, s, r)
    coop.window_search_batched(ss, c, s, r, out, P, n, n)
    torch.cuda.synchronize()
    g = coop.windows_from_device(out)
    del ss, c, s
    o, wall, procs = OP.search_pools(G.MODE_BENCH, 0, p0, P, n)
    for f in ("status", "first", "last", "span", "n_evict"):
        bad = np.nonzero(g[f] != o[f])[0]
        assert bad.size == 0, f"field {f} differs at pools {p0 + bad[:10]}"
    bad = np.nonzero(g["cost"].view(np.uint64) != o["cost"].view(np.uint64))[0]
    assert bad.size == 0, f"cost bits differ at pools {p0 + bad[:10]}"
    st = o["status"]
    assert (st == O.OK).sum() > P * 0.9 and (st == O.INFEASIBLE).sum() > 0
