"""GPU parity of coop_budget_search (waves of coop_replay_trace) with the oracle O4:
minimum and cutoff budgets (values and statuses) on random traces, the Fig. 2 trace and
DNN shapes (R45)."""
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

KEYS = ("peak", "min_budget", "cutoff_budget", "min_status", "cutoff_status")


def same(tr, flags, kc, kf, ctx):
    g = coop.budget_search(coop.Trace(tr), flags, coarse=kc, fine=kf)
    o = O.budget_search(tr, flags, coarse=kc, fine=kf)
    assert {k: int(g[k]) for k in KEYS} == {k: int(o[k]) for k in KEYS}, ctx
    return g


@pytest.mark.parametrize("seed", range(8))
def test_budget_search_random(seed):
    rng = np.random.default_rng(100 + seed)
    tr = TR.random_trace(rng, n_fwd=8 + seed, iters=1 + seed % 2, unit=1 << 10)
    for flags in (0, 1, 2, 3):
        same(tr, flags, 16, 8, f"seed {seed} flags {flags}")


def test_budget_search_fig2():
    g = same(TR.fig2_trace(), 3, 64, 64, "fig2")
    assert g["min_status"] == 0 and g["min_budget"] <= g["cutoff_budget"] <= g["peak"]


@pytest.mark.parametrize("name", ["resnet50", "unet", "swin_t"])
def test_budget_search_dnn(name):
    g = same(dnn.dnn(name), 3, 24, 12, name)
    assert g["min_status"] == 0
