import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from gen import dnn
from paper_2311_00591_b200 import coop
for name, fr in (("resnet50", 0.5),):
    tr = getattr(dnn, name)(); h = coop.Trace(tr); peak = h.peak_live(3)
    out = torch.empty(136, dtype=torch.uint8, device="cuda")
    h.replay_device([int(peak * fr)], 3, out); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): h.replay_device([int(peak * fr)], 3, out)
    e.record(); torch.cuda.synchronize()
    print(name, fr, "ms", round(s.elapsed_time(e) / 5, 3), os.environ.get("COOP_REPLAY_PS"))
