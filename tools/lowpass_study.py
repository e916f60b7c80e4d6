#!/usr/bin/env python
"""NEXT-2: the paper's low-pass DCT optimisation (mode m2 vs m1,
P:118) measured on B200.

On the same UHD 8-bit clips (config 5's segments, G(10 + s)), block 32, the
analyzer runs with the full 32x32 DCT and with the low-pass DCT (2x2 mean, 16x16
DCT, R-5).  Reported per clip:

* throughput of each mode (device-resident frames, CUDA events around
  vca_analyze, best of R repetitions) and the low-pass speed-up;
* agreement of the features between the modes: Pearson correlation over frames
  of E_Y, h and L_Y (the paper's premise: E_Y "exhibits better correlation
  across resolutions"), and the across-clip correlation of the clip means.

Writes one JSON object per clip plus a summary line to stdout.
usage: lowpass_study.py [--clips 8] [--frames 120] [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_12384_b200 import Analyzer, records_to_numpy, synth  # noqa: E402


def timed(a, planes, reps):
    out = torch.empty((planes[0].shape[0], 8), dtype=torch.float64, device="cuda")
    a.reset(0)
    a.analyze(*planes, out=out)
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.reset(0)
        e0.record()
        a.analyze(*planes, out=out)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return records_to_numpy(out), best


def pcc(x, y):
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    if x.std() == 0 or y.std() == 0:
        return float("nan")
    return float(np.corrcoef(x, y)[0, 1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clips", type=int, default=8)
    ap.add_argument("--frames", type=int, default=120)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    W, H = 3840, 2160
    full = Analyzer(W, H, 8, 32, False)
    low = Analyzer(W, H, 8, 32, True)
    means = {"full": [], "low": []}
    rows = []
    for s in range(args.clips):
        planes = synth.g_frames(10 + s, W, H, args.frames, 8, 0, "cuda")
        rf, tf = timed(full, planes, args.reps)
        rl, tl = timed(low, planes, args.reps)
        row = {"clip": "G(%d)" % (10 + s), "frames": args.frames,
               "fps_full": args.frames / tf * 1e3, "fps_lowpass": args.frames / tl * 1e3, "speedup": tf / tl,
               "pcc_E_Y": pcc(rf["E_Y"], rl["E_Y"]), "pcc_h": pcc(rf["h"][1:], rl["h"][1:]),
               "pcc_L_Y": pcc(rf["L_Y"], rl["L_Y"]),
               "mean_E_Y_full": float(rf["E_Y"].mean()), "mean_E_Y_lowpass": float(rl["E_Y"].mean()),
               "ratio_E_Y_low_over_full": float(rl["E_Y"].mean() / rf["E_Y"].mean())}
        rows.append(row)
        means["full"].append(row["mean_E_Y_full"])
        means["low"].append(row["mean_E_Y_lowpass"])
        print(json.dumps(row), flush=True)
        del planes
        torch.cuda.empty_cache()
    summ = {"summary": True, "clips": len(rows),
            "speedup_mean": float(np.mean([r["speedup"] for r in rows])),
            "pcc_E_Y_min": float(np.min([r["pcc_E_Y"] for r in rows])),
            "pcc_h_min": float(np.nanmin([r["pcc_h"] for r in rows])),
            "pcc_clip_mean_E_Y": pcc(means["full"], means["low"]) if len(rows) > 2 else None}
    print(json.dumps(summ), flush=True)


if __name__ == "__main__":
    main()
