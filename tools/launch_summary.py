"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import collections, csv, io, sys
path, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
text = open(path).read()
text = text[text.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(text)))
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    ms = v / 1e6 if unit == "nsecond" else v / 1e3 if unit == "usecond" else v if unit == "msecond" else v / 1e6
    name = r["Kernel Name"].split("(")[0]
    tot[name] += ms
    cnt[name] += 1
all_ms = sum(tot.values())
lines = ["# launch list (ncu --metrics gpu__time_duration.sum --clock-control none) of:",
         f"#   {cmd}",
         "# cold-cache, serialised per-launch times: compare shares, not absolutes",
         f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    lines.append(f"{k[:70]:70s} {cnt[k]:8d} {v:10.2f} {v / all_ms * 100:6.1f}%")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
