#!/usr/bin/env python
"""Throughput of every BASELINE.json config on one GPU (device-resident frames,
CUDA events around vca_analyze; block-kernel time from the library's events)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2304_12384_b200 import Analyzer, synth  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
for cfg in (int(x) for x in (sys.argv[1:] or ["1", "2", "3", "4"])):
    c = synth.CONFIGS[cfg]
    F = min(c.n_frames, 600)
    Y, U, V = synth.config_frames(cfg, device="cuda", n_frames=F)
    fb = (c.width * c.height + 2 * (c.width // 2) * (c.height // 2)) * (1 if c.bit_depth == 8 else 2)
    a = Analyzer(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
    steps = 20 if F * fb > 1e9 else 200
    for _ in range(3):
        a.reset(0)
        a.analyze(Y, U, V)
    torch.cuda.synchronize()
    a.profile_read()
    a.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        a.reset(0)
        a.analyze(Y, U, V)
    e1.record()
    torch.cuda.synchronize()
    blk, fin, n = a.profile_read()
    ms = e0.elapsed_time(e1) / steps
    gbs = F * fb / (blk / steps) / 1e6
    print(json.dumps({"config": cfg, "name": c.name, "frames": F, "path": a.info["path"], "ms_per_call": ms,
                      "fps": F / ms * 1e3, "block_kernel_GBps": gbs, "roofline_frac": gbs / peak,
                      "roofline_fps": peak * 1e9 / fb, "in_L2": F * fb < 100e6}), flush=True)
