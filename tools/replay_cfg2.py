import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from gen import dnn
from paper_2311_00591_b200 import coop
tr = dnn.resnet50(); h = coop.Trace(tr); peak = h.peak_live(3)
out = torch.empty(136, dtype=torch.uint8, device="cuda")
for _ in range(2):
    h.replay_device([peak // 2], 3, out); torch.cuda.synchronize()
