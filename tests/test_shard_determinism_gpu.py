"""Determinism across the number of GPUs G ("results must be byte-identical
for every G"), on one GPU: the shards that G ranks would own are run one after another
(their own launches, grids and pool counts) with the same sharding helpers bench.py uses
(dist.pool_range / dist.cyclic_cells) and reassembled with the gather's own assembly
(dist.assemble_cyclic); the bytes must equal the G = 1 run's."""
import numpy as np
import pytest

from gen import dnn
from gen import pools as G

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2311_00591_b200 import coop  # noqa: E402
from paper_2311_00591_b200 import dist as D  # noqa: E402

DEV = torch.device("cuda:0")


def search_shard(p0, P, n=4096):
    ss = torch.empty(P * n, dtype=torch.int64, device=DEV)
    c = torch.empty(P * n, dtype=torch.float64, device=DEV)
    s = torch.empty(P * n, dtype=torch.float64, device=DEV)
    r = torch.empty(P, dtype=torch.int64, device=DEV)
    out = torch.empty(P * 4, dtype=torch.int64, device=DEV)
    G.bench_pools_device(G.MODE_BENCH, 0, p0, P, n, n, ss, c, s, r)
    coop.window_search_batched(ss, c, s, r, out, P, n, n)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint8).copy()


def test_search_shards_byte_identical_for_g_1_2_4_8():
    total = 4096  # pools (strong split of one global set)
    ref = search_shard(0, total)
    for g in (2, 4, 8):
        per = total // g
        parts = [search_shard(D.pool_range(per, r)[0], per) for r in range(g)]
        assert np.concatenate(parts).tobytes() == ref.tobytes(), f"G = {g}"


def test_replay_cells_byte_identical_for_g_1_2_4_8():
    """BASELINE config 3 (GPT-3-style 2.7B x 64 budgets), cells cyclic over ranks."""
    flags = coop.F_PARTITION | coop.F_INPLACE
    t = coop.Trace(dnn.gpt3_2p7b())
    peak = t.peak_live(flags)
    budgets = [peak * (1575 + 75 * k) // 6300 for k in range(64)]
    ref, _ = t.replay(budgets, flags)
    for g in (2, 4, 8):
        parts = []
        for r in range(g):
            mine = D.cyclic_cells(len(budgets), r, g)
            res, _ = t.replay([budgets[c] for c in mine], flags)
            parts.append(res)
        got = D.assemble_cyclic(parts, len(budgets), g)
        # every field but the wall-clock search latency (not bit-exact by definition, R28)
        keep = [f for f in ref.dtype.names if not f.startswith("search_ns")]
        for f in keep:
            assert np.array_equal(got[f], ref[f]), f"G = {g} field {f}"
    t.close()
