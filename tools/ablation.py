"""App. B ablation on the synthetic DNN traces, through
coop_replay_trace / coop_budget_search on the GPU:

  full          Coop: sliding window + partitioning + recomputable in-place (P|I)
  no-window     DTE's heuristic loop instead of the sliding window, P|I kept
  no-inplace    copy-on-write instead of recomputable in-place (P)
  no-partition  every tensor placed from the left (I)

Budgets are fractions of ONE common peak (the full variant's R25 peak), so every variant
gets the same bytes at a given memory ratio.  Per (variant, ratio): completed or OOM,
compute overhead (total - base) / base, fragmentation rate (R27); per variant the minimum
budget (R45 grid search) as a fraction of that peak.  Directions to compare with the
paper: removing any module raises the lowest budget (ResNet-50: 30 % -> 40 %), and the
sliding window matters most for overhead (U-Net at 40 %: ~2x without it)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from gen import dnn  # noqa: E402
from paper_2311_00591_b200 import coop  # noqa: E402

P, I = coop.F_PARTITION, coop.F_INPLACE
VARIANTS = {"full": P | I, "no-window": coop.F_POLICY_DTE | P | I, "no-inplace": P, "no-partition": I}
RATIOS = [r / 100 for r in range(20, 101, 10)]


def main(names):
    for name in names:
        tr = coop.Trace(dnn.dnn(name))
        peak = tr.peak_live(P | I)
        print(f"== {name}: common peak {peak / 2**20:.1f} MiB (full variant, R25)")
        print("variant       min-budget  " + "  ".join(f"{int(r * 100):>11d}%" for r in RATIOS))
        for v, flags in VARIANTS.items():
            bs = coop.budget_search(tr, flags, coarse=40, fine=20)
            mb = f"{bs['min_budget'] / peak:9.3f}" if bs["min_status"] == 0 else "      OOM"
            res, _ = tr.replay([int(peak * r) for r in RATIOS], flags)
            cells = []
            for r in res:
                if r["status"] != 0:
                    cells.append("        OOM")
                else:
                    ov = (r["total_us"] - r["base_us"]) / max(1, r["base_us"])
                    fr = r["sum_free_bytes_after"] / max(1, r["pressure"] * r["budget"])
                    cells.append(f"{ov:5.2f}/{fr:5.3f}")
            print(f"{v:13s} {mb}  " + "  ".join(cells))
        print("(cells: overhead / fragmentation rate; min-budget: fraction of the common peak)")
        tr.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["resnet50", "unet", "swin_t", "bert_large", "inception_v3"])
