import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2304_12384_b200 import Analyzer, synth
W, H, w, lp = int(os.environ["PW"]), int(os.environ["PH"]), int(os.environ["PB"]), bool(int(os.environ["PL"]))
Y, U, V = synth.g_frames(7, W, H, 120, 8, 0, "cuda")
a = Analyzer(W, H, 8, w, lp)
for _ in range(3):
    a.reset(0); a.analyze(Y, U, V)
torch.cuda.synchronize(); print("ok", a.info["path"])
