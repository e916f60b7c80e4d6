#!/usr/bin/env python
"""Small driver for ncu captures: analyse PROF_FRAMES frames of a config a few
times (the last launch is the one to capture with -s/-c)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2304_12384_b200 import Analyzer, synth  # noqa: E402

cfg = int(os.environ.get("PROF_CONFIG", "3"))
F = int(os.environ.get("PROF_FRAMES", "120"))
reps = int(os.environ.get("PROF_REPS", "3"))
c = synth.CONFIGS[cfg]
Y, U, V = synth.config_frames(cfg, device="cuda", n_frames=F)
a = Analyzer(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
for _ in range(reps):
    a.reset(0)
    a.analyze(Y, U, V)
torch.cuda.synchronize()
print("ok", cfg, F, reps)
