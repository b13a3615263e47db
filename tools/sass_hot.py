"""Summarise an ncu --page source --print-source sass CSV: hottest SASS by samples / executed,
with source lines mapped through nvdisasm -g line info of the given cubin/.so (optional)."""
import csv, sys, re, subprocess, collections
path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def f(r, k):
    try: return float(r[idx[k]].replace(',', ''))
    except: return 0.0
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_e = sum(f(r, "Instructions Executed") for r in data)
print("total samples", tot_s, "total warp-inst executed", tot_e)
# optional line map
linemap = {}
if len(sys.argv) > 2:
    out = subprocess.run(["cuobjdump", "-sass", "-fun", sys.argv[3], sys.argv[2]] if len(sys.argv) > 3 else ["true"], capture_output=True, text=True).stdout
key = sys.argv[4] if len(sys.argv) > 4 else None
top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:40]
for r in top:
    print(f"{r[idx['Address']]:>8} {f(r,'Warp Stall Sampling (All Samples)')/tot_s*100:5.1f}% exec {f(r,'Instructions Executed')/tot_e*100:5.2f}%  {r[idx['Source']][:90]}")
