"""Map an ncu SASS source-page CSV onto CUDA source lines via nvdisasm -g line info.
usage: [SORT=stall] sass_lines.py <ncu_sass.csv> <lib.so> <kernel-substring> [top]"""
import collections, csv, os, re, subprocess, sys, tempfile

csv_path, lib, ksub = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def f(r, k):
    try: return float(r[idx[k]].replace(',', ''))
    except Exception: return 0.0
base = int(data[0][idx["Address"]], 16)

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
fns = set()
for cub in os.listdir(tmp):
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    cur_fn, cur_line, cur_file = None, None, None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln) or re.match(r"^(\S+):\s*$", ln)
        if ln.startswith(".text.") or re.match(r"^\s*\.section\s+\.text\.", ln):
            pass
        m = re.search(r"\.text\.([A-Za-z0-9_]+)", ln)
        if m and ("section" in ln):
            cur_fn = m.group(1)
            if ksub in cur_fn:
                fns.add(cur_fn)
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_file, cur_line = os.path.basename(m.group(1)), int(m.group(2))
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and ksub in cur_fn:
            line_of[int(m.group(1), 16)] = (cur_file, cur_line)
if len(fns) > 1:
    sys.exit("kernel substring matches several functions (pass e.g. search_kernelILi8ELi512ELi1E):\n  "
             + "\n  ".join(sorted(fns)))
agg_e = collections.Counter(); agg_s = collections.Counter()
tot_e = tot_s = 0
for r in data:
    off = int(r[idx["Address"]], 16) - base
    key = line_of.get(off, ("?", 0))
    e = f(r, "Instructions Executed"); s = f(r, "Warp Stall Sampling (All Samples)")
    agg_e[key] += e; agg_s[key] += s; tot_e += e; tot_s += s
print(f"mapped {len(line_of)} offsets; total exec {tot_e:.3g} samples {tot_s:.3g}")
src_cache = {}
def src(fn, l):
    for root in ("paper_2311_00591_b200/csrc", "."):
        p = os.path.join(root, fn)
        if os.path.exists(p):
            src_cache.setdefault(p, open(p).read().splitlines())
            L = src_cache[p]
            return L[l - 1].strip()[:70] if 0 < l <= len(L) else ""
    return ""
by_stall = os.environ.get("SORT") == "stall"
print("--- by " + ("warp stall samples" if by_stall else "executed instructions"))
for k, v in (agg_s if by_stall else agg_e).most_common(top):
    print(f"{agg_e[k] / tot_e * 100:5.1f}% exec {agg_s[k] / tot_s * 100:5.1f}% stall  {k[0]}:{k[1]}  {src(*k)}")

if os.environ.get("RANGES"):
    print("--- by line range")
    for spec in os.environ["RANGES"].split(";"):
        name, rng = spec.split("=")
        lo, hi = map(int, rng.split("-"))
        e = sum(v for k, v in agg_e.items() if k[0] == "coop_search.cu" and lo <= k[1] <= hi)
        st = sum(v for k, v in agg_s.items() if k[0] == "coop_search.cu" and lo <= k[1] <= hi)
        print(f"{name:>12}: exec {e / tot_e * 100:5.1f}%  stall {st / tot_s * 100:5.1f}%")
    oth = sum(v for k, v in agg_e.items() if k[0] != "coop_search.cu")
    print(f"{'other files':>12}: exec {oth / tot_e * 100:5.1f}%")
