#!/usr/bin/env python
"""Throughput of every (block size, low-pass) family the API accepts, on 1080p and UHD
8-bit synthetic frames (device-resident, CUDA events): which kernel path each uses and how
fast it is relative to the HBM roofline."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2304_12384_b200 import Analyzer, synth  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
for (W, H, F) in ((1920, 1080, 120), (3840, 2160, 60), (1280, 720, 240)):
    Y, U, V = synth.g_frames(7, W, H, F, 8, 0, "cuda")
    fb = W * H * 3 // 2
    for (w, lp) in ((0, False), (0, True), (4, False), (8, False), (16, False), (16, True), (32, False), (32, True)):
        try:
            a = Analyzer(W, H, 8, w, lp)
        except Exception as e:
            print(json.dumps({"W": W, "H": H, "w": w, "lowpass": lp, "error": str(e)}))
            continue
        for _ in range(2):
            a.reset(0)
            a.analyze(Y, U, V)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            a.reset(0)
            a.analyze(Y, U, V)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"W": W, "H": H, "block": a.info["block"][0], "lowpass": lp, "path": a.info["path"],
                          "fps": round(F / ms * 1e3), "roofline_frac": round(F * fb / (ms / 1e3) / 1e9 / peak, 3)}),
              flush=True)
