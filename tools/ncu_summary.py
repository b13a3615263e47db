"""Summarise an ncu report (--set full) into a small text file for profiles/."""
import csv, io, subprocess, sys
rep, out_path, label = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
        "sm__cycles_elapsed.avg"]
lines = [f"# {label}", f"# source: {rep} (ncu --set full --clock-control none)"]
for r in rows[2:]:
    d = dict(zip(h, r))
    un = dict(zip(h, u))
    for k in keys:
        if k in d:
            lines.append(f"{k} = {d[k]} {un.get(k, '')}".rstrip())
    st = sorted([(k, d[k]) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k],
                key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
    lines.append("top stall reasons (pc samples):")
    for k, v in st:
        lines.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} = {v}")
open(out_path, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
