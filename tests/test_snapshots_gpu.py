"""The replay-snapshot workload of config 4 (the item list of PAPER.md:147):
coop_replay_snapshots records the item view of every Coop pressure event of a GPU replay;
coop_window_search_batched on those rows must return exactly the window the replay evicted,
and the O1 oracle on the same rows must agree bit for bit.  The replay itself is bit-exact
with O2 (counters, digest), so the recorded windows are the ones Alg. 1 evicts."""
import numpy as np
import pytest

from gen import dnn
from gen import traces as TR
from oracle import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2311_00591_b200 import coop  # noqa: E402

FIELDS = ("status", "first", "last", "span", "n_evict")


def check(tr, frac, n_max, cap, flags=coop.F_PARTITION | coop.F_INPLACE):
    t = coop.Trace(tr)
    budget = int(t.peak_live(flags) * frac)
    d = t.snapshots(budget, flags, n_max, cap)
    want_r, _ = O.replay(tr, budget, flags)
    r = d["result"]
    for f in ("status", "evictions", "pressure", "remat", "digest", "heuristic_evals"):
        assert int(r[f]) == int(want_r[f]), f
    k = d["count"]
    assert k == min(cap, int(r["pressure"])) or int(r["max_blocks"]) > n_max
    if k == 0:
        return 0
    rec = coop.windows_from_device(d["windows"][:4 * k])
    out = torch.empty(k * 4, dtype=torch.int64, device="cuda")
    coop.window_search_batched(d["ss"], d["cost"], d["stale"], d["requests"], out, k, n_max, n_max)
    torch.cuda.synchronize()
    g = coop.windows_from_device(out)
    for f in FIELDS:
        assert np.array_equal(g[f], rec[f]), f
    assert np.array_equal(g["cost"].view(np.uint64), rec["cost"].view(np.uint64))
    ss = d["ss"][:k * n_max].cpu().numpy().view(np.uint64)
    o = O.search_many(ss, d["cost"][:k * n_max].cpu().numpy(), d["stale"][:k * n_max].cpu().numpy(),
                      d["requests"][:k].cpu().numpy().view(np.uint64), k, n_max, n_max)
    for f in FIELDS:
        assert np.array_equal(o[f], rec[f]), f
    assert np.array_equal(o["cost"].view(np.uint64), rec["cost"].view(np.uint64))
    t.close()
    return k


@pytest.mark.parametrize("name,frac", [("resnet50", 0.5), ("gpt3_2.7b", 0.6), ("unet", 0.55),
                                       ("bert_large", 0.4), ("inception_v3", 0.35)])
def test_snapshots_dnn(name, frac):
    assert check(dnn.dnn(name), frac, 4096, 4096) > 10


def test_snapshots_fig2_and_small_rows():
    assert check(TR.fig2_trace(), 0.7, 16, 8, flags=0) > 0
    k = check(dnn.resnet50(), 0.45, 1024, 100000)
    assert k > 0


def test_snapshots_invalid_args():
    t = coop.Trace(TR.fig2_trace())
    with pytest.raises(coop.CoopError):
        t.snapshots(250 << 20, coop.F_POLICY_DTR, 16, 4)
    with pytest.raises(coop.CoopError):
        t.snapshots(250 << 20, 0, 0, 4)
