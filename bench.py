#!/usr/bin/env python
"""bench.py -- Coop window-search benchmark (BASELINE.json config 4) on 1..8 B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl coop|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...       (one rank per GPU, NCCL)

A "step" is one pass of the batched search hot path (load the SoA
block tables, h = c/s, span/cost prefix scans, per-start window ends, argmin, exact verify,
output) over the rank's whole shard: 2^20 pools x 4096 blocks per GPU (weak scaling: each
rank owns the pools [rank * 2^20, (rank + 1) * 2^20) of the global counter-based sequence
and generates them on its own device, untimed; no data-path collective).  Inputs are
96 GiB per GPU >> 126 MB L2, so no L2 flush is needed between steps.

Rank 0 prints ONE JSON line.  `value` = pools searched per second over all ranks
(max-over-ranks device time); `roofline` = algorithmic HBM bytes per launch / measured
kernel time vs MEASURED_PEAKS.json; `cpu_baseline` = the CPU oracle (oracle/) timed on this
box's host cores on a bounded sample; `e2e` = the same metric through the host-buffer C-ABI
entry point (coop_window_search_batched_host) with H2D/D2H copies inside the timed region.
`--impl reference` times the oracle itself (rank 0 only) on bounded samples per step.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_BLOCKS = 4096
POOLS_PER_GPU = 1 << 20
ALGO_BYTES_PER_POOL = 24 * N_BLOCKS + 8 + 32  # size_state+cost+stale, request, result
SEED = 0
METRIC = "window-search queries/s"
UNIT = "queries/s"
ARM_CONFIG = {"workload": "config4: batched window search, 2^20 pools x 4096 blocks per GPU "
                          "(BASELINE.json configs[3])",
              "pools_per_gpu": POOLS_PER_GPU, "n_blocks": N_BLOCKS, "seed": SEED,
              "l2": "no flush: 96 GiB of inputs per step per GPU >> 126 MB L2",
              "generator": "gen/coop_gen.cu MODE_BENCH (counter-based)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="coop", choices=["coop", "reference"])
    ap.add_argument("--pools", type=int, default=POOLS_PER_GPU, help="pools per GPU")
    ap.add_argument("--e2e-pools", type=int, default=65536)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-replay", action="store_true", help="skip the replay sweeps")
    ap.add_argument("--replay-steps", type=int, default=2)
    ap.add_argument("--no-config5", action="store_true",
                    help="skip config 5 (8 DNN shapes x 256 budgets; ~2 min on one B200)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="CPU work budget of the oracle baseline sample")
    return ap.parse_args()


# ----------------------------------------------------------------------------- peaks
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the search kernel from the committed ncu --set full capture"""
    p = os.path.join(ROOT, "profiles", "search_ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d
    return None


# ----------------------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
                power.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------- oracle baseline
def _oracle_worker(args):
    """Runs in a worker process: generate a contiguous slice of the workload's pools on the
    host, wait for all workers, then time the oracle on it."""
    p0, n_pools, barrier = args
    from gen import pools as G
    from oracle import oracle as O
    ss, c, s, r = G.bench_pools_host(G.MODE_BENCH, SEED, p0, n_pools, N_BLOCKS)
    barrier.wait()
    t = time.perf_counter()
    O.search_many(ss, c, s, r, n_pools, N_BLOCKS, N_BLOCKS)
    return n_pools, time.perf_counter() - t


def cpu_baseline(cpu_seconds: float, sample_offset: int = 0):
    cores = os.cpu_count() or 1
    per_pool_s = 0.004  # oracle ~4 ms per 4096-block pool (one core), to size the sample
    per_worker = max(2, int(cpu_seconds / per_pool_s / cores))
    per_worker += per_worker % 2  # even: short and long requests alike
    ctx = mp.get_context("fork")
    with ctx.Manager() as m:
        barrier = m.Barrier(cores)
        with ctx.Pool(cores) as pool:
            res = pool.map(_oracle_worker, [(sample_offset + w * per_worker, per_worker, barrier)
                                            for w in range(cores)])
    total = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"value": total / wall, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{total} pools x {N_BLOCKS} blocks (global pools "
                      f"[{sample_offset}, {sample_offset + total})), one process per core, "
                      f"C oracle O(N*L) per pool, wall {wall:.2f} s"}


# ------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    per_worker = 16  # ~60 ms of oracle work per worker per step (bounded sample)
    ctx = mp.get_context("fork")
    times = []
    total = 0
    with ctx.Manager() as m:
        with ctx.Pool(cores) as pool:
            for step in range(args.warmup + args.steps):
                barrier = m.Barrier(cores)
                off = step * cores * per_worker
                res = pool.map(_oracle_worker, [(off + w * per_worker, per_worker, barrier)
                                                for w in range(cores)])
                if step >= args.warmup:
                    times.append(max(r[1] for r in res))
                    total += sum(r[0] for r in res)
    t = sum(times)
    value = total / t
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(ARM_CONFIG, sample=f"bounded sample per step: {cores * per_worker} "
                                                   f"pools of the same workload (global pools from 0)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{cores * per_worker} pools per step, one process per core"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------- replay sweeps
def replay_bench(world: int, rank: int, steps: int, with_config5: bool):
    """BASELINE configs 3 and 5 on this rank's cells (config 5 cells cyclic over ranks):
    trace ops/s = trace ops (not counting recomputes) replayed per second, summed over
    cells; device time per sweep with CUDA events; one stream per trace."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from gen import dnn
    from paper_2311_00591_b200 import coop
    from paper_2311_00591_b200 import dist as D

    flags = coop.F_PARTITION | coop.F_INPLACE
    out = {}
    traces = {name: dnn.dnn(name) for name in dnn.DNNS}
    handles = {name: coop.Trace(tr) for name, tr in traces.items()}
    peaks = {name: handles[name].peak_live(flags) for name in traces}
    sweeps = {
        # config 2: ResNet-50 at 50 % of peak, one cell
        "config2": [("resnet50", [peaks["resnet50"] // 2])],
        # config 3: GPT-3-style 2.7B, 64 budgets 25 %..100 % of peak, one CTA per budget
        "config3": [("gpt3_2.7b", [peaks["gpt3_2.7b"] * (1575 + 75 * k) // 6300 for k in range(64)])],
        # config 5: eight DNN shapes x 256 budgets 20 %..100 % of peak
        "config5": [(name, [peaks[name] * (20 * 255 + 80 * k) // (100 * 255) for k in range(256)])
                    for name in dnn.DNNS],
    }
    if not with_config5:
        del sweeps["config5"]
    streams = {name: torch.cuda.Stream() for name in traces}
    main_s = torch.cuda.current_stream()
    for key, sweep in sweeps.items():
        # shard: global cell index over the sweep, cyclic over ranks (config 3 too)
        cells = [(name, j, b) for name, bs in sweep for j, b in enumerate(bs)]
        mine = [cells[c] for c in D.cyclic_cells(len(cells), rank, world)]
        per = {}
        for name, j, b in mine:
            per.setdefault(name, []).append(b)
        bufs = {name: torch.empty(len(bs) * coop.REPLAY_RESULT_DTYPE.itemsize, dtype=torch.uint8,
                                  device="cuda") for name, bs in per.items()}
        ops = sum(traces[name].n_ops * len(bs) for name, bs in per.items())

        def sweep_once(warm=False):
            ev0 = torch.cuda.Event()
            ev0.record(main_s)
            for name, bs in per.items():
                st = streams[name]
                st.wait_event(ev0)
                # warm-up: the same cell count at the peak budget (no pressure: cheap), which
                # allocates the per-trace workspaces outside the timed region
                handles[name].replay_device([peaks[name]] * len(bs) if warm else bs, flags,
                                            bufs[name], stream=st)
            for name in per:
                e = torch.cuda.Event()
                e.record(streams[name])
                main_s.wait_event(e)

        sweep_once(warm=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        nsteps = 1 if key == "config5" else steps  # config 5: one sweep takes minutes
        t0.record(main_s)
        for _ in range(nsteps):
            sweep_once()
        t1.record(main_s)
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / nsteps
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t[0])
            tops = torch.tensor([ops], dtype=torch.float64, device="cuda")
            dist.all_reduce(tops)
            ops_all = float(tops[0])
        else:
            ops_all = float(ops)
        res = np.concatenate([bufs[n].cpu().numpy().view(coop.REPLAY_RESULT_DTYPE) for n in per]) \
            if per else np.zeros(0, coop.REPLAY_RESULT_DTYPE)
        ok = res["status"] == 0
        frag = (res["sum_free_bytes_after"][ok] / np.maximum(1, res["pressure"][ok]) /
                res["budget"][ok].astype(np.float64))
        ovh = (res["total_us"][ok] - res["base_us"][ok]) / np.maximum(1, res["base_us"][ok])
        lat = res["search_ns_total"][ok] / np.maximum(1, res["pressure"][ok])
        out[key] = {
            "workload": {"config2": "ResNet-50 at 50 % of peak, 1 budget",
                         "config3": "GPT-3-style 2.7B x 64 budgets (25-100 % of peak)",
                         "config5": "8 DNN shapes x 256 budgets (20-100 % of peak)"}[key],
            "flags": "partition+recomputable-inplace", "cells": len(cells),
            "cells_this_rank": len(mine), "ms_per_sweep": ms, "timed_sweeps": nsteps,
            "trace_ops_per_s": ops_all / (ms / 1e3),
            "events_per_s_incl_recompute": (ops_all + float(res["remat"].sum()) * world) / (ms / 1e3),
            "completed_cells_rank0": int(ok.sum()),
            "mean_frag_rate_rank0": float(frag.mean()) if ok.any() else None,
            "mean_overhead_rank0": float(ovh.mean()) if ok.any() else None,
            "search_latency_us_mean_rank0": float(lat.mean() / 1e3) if ok.any() else None,
            "search_latency_us_max_rank0": float(res["search_ns_max"][ok].max() / 1e3) if ok.any() else None,
            "gpu_launches_per_sweep": len(per),
        }
    # NEXT-3: minimum / cutoff budgets (R45) of the config-2 and config-3 traces, rank 0 only
    if rank == 0:
        for name in ("resnet50", "gpt3_2.7b"):
            t0 = time.perf_counter()
            b = coop.budget_search(handles[name], flags, coarse=64, fine=64)
            dt = time.perf_counter() - t0
            pk = float(b["peak"])
            out.setdefault("budgets", {})[name] = {
                "peak_bytes": int(b["peak"]),
                "min_budget_frac": (int(b["min_budget"]) / pk) if b["min_status"] == 0 else None,
                "cutoff_budget_frac": (int(b["cutoff_budget"]) / pk) if b["cutoff_status"] == 0 else None,
                "replays": int(b["replays"]), "wall_ms": dt * 1e3,
                "grid": "64 coarse x 64 fine budgets (DESIGN.md R45)"}
    for h in handles.values():
        h.close()
    return out


# ---------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from gen import pools as G
    from paper_2311_00591_b200 import coop

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    P, n = args.pools, N_BLOCKS
    p0 = rank * P
    ss = torch.empty(P * n, dtype=torch.int64, device=dev)
    c = torch.empty(P * n, dtype=torch.float64, device=dev)
    s = torch.empty(P * n, dtype=torch.float64, device=dev)
    r = torch.empty(P, dtype=torch.int64, device=dev)
    out = torch.empty(P * 4, dtype=torch.int64, device=dev)
    G.bench_pools_device(G.MODE_BENCH, SEED, p0, P, n, n, ss, c, s, r)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()

    def step():
        coop.window_search_batched(ss, c, s, r, out, P, n, n, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t_all0 = torch.cuda.Event(enable_timing=True)
    t_all1 = torch.cuda.Event(enable_timing=True)
    t_all0.record(stream)
    for e0, e1 in evs:
        e0.record(stream)
        step()
        e1.record(stream)
    t_all1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()

    elapsed_ms = t_all0.elapsed_time(t_all1)
    kernel_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    if world > 1:
        t = torch.tensor([elapsed_ms, statistics.mean(kernel_ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, kmean = float(t[0]), float(t[1])
    else:
        kmean = statistics.mean(kernel_ms)

    # results summary (untimed): status histogram; gather per-rank digests to rank 0
    res = coop.windows_from_device(out)
    digest = int(np.bitwise_xor.reduce(res.view(np.uint64)))
    stat = {str(k): int(v) for k, v in zip(*np.unique(res["status"], return_counts=True))}
    if world > 1:
        # the path's only collective: gather of per-shard results (here: shard digests)
        d = torch.tensor([digest & 0x7FFFFFFFFFFFFFFF], dtype=torch.int64, device=dev)
        gathered = [torch.zeros_like(d) for _ in range(world)]
        dist.all_gather(gathered, d)

    # e2e through the host-buffer C-ABI entry (rank-local; pinned host copies, untimed fill)
    e2e = None
    Pe = min(args.e2e_pools, P)
    if Pe > 0:
        h_ss = torch.empty(Pe * n, dtype=torch.int64, pin_memory=True)
        h_c = torch.empty(Pe * n, dtype=torch.float64, pin_memory=True)
        h_s = torch.empty(Pe * n, dtype=torch.float64, pin_memory=True)
        h_r = torch.empty(Pe, dtype=torch.int64, pin_memory=True)
        h_ss.copy_(ss[:Pe * n]); h_c.copy_(c[:Pe * n]); h_s.copy_(s[:Pe * n]); h_r.copy_(r[:Pe])
        h_out = np.empty(Pe, dtype=coop.WINDOW_DTYPE)
        coop.window_search_batched_host(h_ss, h_c, h_s, h_r, Pe, n, n, out=h_out)  # warm-up
        k_e2e = 3
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            coop.window_search_batched_host(h_ss, h_c, h_s, h_r, Pe, n, n, out=h_out)
        te = (time.perf_counter() - t0) / k_e2e
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        same = h_out.tobytes() == res[:Pe].tobytes()
        e2e = {"value": world * Pe / te, "unit": UNIT,
               "h2d_bytes_per_step": Pe * n * 24 + Pe * 8, "d2h_bytes_per_step": Pe * 32,
               "pools_per_gpu": Pe, "matches_device_results": same,
               "api": "coop_window_search_batched_host (pinned host buffers, chunked "
                      "H2D/kernel/D2H overlap on 2 streams)"}
        del h_ss, h_c, h_s, h_r

    value = world * P * args.steps / (elapsed_ms / 1e3)
    peak, peak_src = peaks()
    achieved = P * ALGO_BYTES_PER_POOL / (kmean / 1e3) / 1e9
    tr = ncu_traffic()
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_src,
            "traffic": (tr["dram_bytes_per_pool"] * P) if tr else None,
            "algorithmic_bytes_per_launch": P * ALGO_BYTES_PER_POOL,
            "kernel": "coop::search_kernel<8,512,2>", "kernel_ms_mean": kmean,
            "frac_of_8TBps": achieved / 8000.0}
    replay = None
    if not args.no_replay:
        replay = replay_bench(world, rank, args.replay_steps, not args.no_config5)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_seconds)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(ARM_CONFIG, pools_per_gpu=P,
                               parallelism=f"dp{world} (pool shards, weak scaling)"),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": args.steps, "clocks": clk, "replay": replay,
                "results": {"status_counts": stat, "xor_digest": f"{digest:016x}"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
