#!/usr/bin/env python
"""NEXT-2: the paper's low-pass optimisation and the cross-resolution stability of
E_Y, measured on B200 with the HEAD build, to SPEC's acceptance criteria 6 and 8
(the paper: "spatially downsampled by a factor of two",
P:118 m2 vs m1).

Corpora: >= 20 seeded synthetic clips each, rendered at 2160p and area-downsampled (2x2 / 4x4
box mean, rounded) to 1080p and 540p -- the same content at three resolutions, as an encoding
ladder would have it: "g" = generator G(seed) of BASELINE.json config 2 (three moving oriented
tones + strong white noise, scene cuts), and "pink" = a 1/f^beta spectrum (8 moving tones with
amplitude growing with wavelength, mild noise; see pink_frames), closer to the statistics of
natural video.  Both stand in for the paper's unnamed UHD videos; nothing here is
from a dataset.

Per clip:
  * fps of the full 32x32 DCT and of the low-pass DCT (2x2 mean + 16x16 DCT) at 2160p, same
    device-resident frames, CUDA events around vca_analyze, best of --reps;
  * mean E_Y at 2160p full, 2160p low-pass, 1080p and 540p (block size by the auto rule S:250:
    32 / 16 / 8, full DCT), plus per-frame PCC of E_Y low-pass vs full.
Summary (the acceptance numbers):
  * speedup = fps(low-pass) / fps(full)   (criterion 8: >= 1.8)
  * PCC over clips of mean E_Y, low-pass vs full at 2160p   (criterion 8: >= 0.90)
  * PCC over clips of mean E_Y across resolution pairs 2160/1080, 2160/540, 1080/540
    (criterion 6: >= 0.90; its SI comparison is out of scope -- SI/TI is the paper's comparison
    system).
usage: lowpass_study.py [--clips 24] [--frames 48] [--reps 5] [--out FILE]
"""
import argparse
import json
import math
import os
import subprocess
import sys
import time

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


def pink_frames(seed, W, H, F, device="cuda"):
    """A second corpus with a natural-image-like 1/f^beta spectrum (input rendering only): per
    clip and plane, 8 moving oriented sinusoids with wavelengths log-uniform in [4, 512] px and
    amplitude a0 (lambda / 64)^beta (beta ~ U[0.5, 1.5], a0 log-uniform in [2, 60]), plus mild
    white noise sigma ~ U[0.5, 2]; uint8.  Unlike G(seed) -- three tones of equal weight plus
    strong white noise, all clips of similar complexity -- its energy is spread across scales
    the way natural video's is, and its clips span a wide complexity range (flat to busy), as a
    real corpus does."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 7])))
    dims = ((W, H), (W // 2, H // 2), (W // 2, H // 2))
    out = tuple(torch.empty((F, h, w), dtype=torch.uint8, device=device) for (w, h) in dims)
    beta, a0 = rng.uniform(0.5, 1.5), math.exp(rng.uniform(math.log(2.0), math.log(60.0)))
    planes = []
    for p, (w, h) in enumerate(dims):
        sc = 1.0 if p == 0 else 0.5
        sines = []
        for _ in range(8):
            lam = math.exp(rng.uniform(math.log(4.0), math.log(512.0)))
            sines.append((rng.uniform(0, math.pi), lam * sc, a0 * (lam / 64.0) ** beta / 3.0, rng.uniform(0, 2 * math.pi),
                          rng.uniform(0.0, 3.0) * sc))
        planes.append((sines, rng.uniform(0.5, 2.0)))
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    for t in range(F):
        for p, (w, h) in enumerate(dims):
            y = torch.arange(h, device=device, dtype=torch.float64).view(h, 1)
            x = torch.arange(w, device=device, dtype=torch.float64).view(1, w)
            v = torch.full((h, w), 128.0, dtype=torch.float64, device=device)
            sines, sigma = planes[p]
            for (th, lam, A, ph, vel) in sines:
                v += A * torch.sin(x * (2 * math.pi * math.cos(th) / lam) + y * (2 * math.pi * math.sin(th) / lam)
                                   + (ph - 2 * math.pi * vel * t / lam))
            v += sigma * torch.randn((h, w), generator=g, device=device, dtype=torch.float64)
            out[p][t] = torch.clamp(torch.round(v), 0, 255).to(torch.uint8)
    return out


def downsample(planes, f):
    """Area (f x f box mean, rounded half to even) downsampling of uint8 planes: input rendering."""
    res = []
    for p in planes:
        q = torch.nn.functional.avg_pool2d(p.float().unsqueeze(1), f).squeeze(1)
        res.append(torch.round(q).clamp(0, 255).to(torch.uint8).contiguous())
    return tuple(res)


def pcc(x, y):
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    if len(x) < 3 or x.std() == 0 or y.std() == 0:
        return float("nan")
    return float(np.corrcoef(x, y)[0, 1])


def study(corpus, args, an):
    W, H = 3840, 2160
    rows = []
    for s in range(args.clips):
        seed = args.first_seed + s
        uhd = (synth.g_frames(seed, W, H, args.frames, 8, 0, "cuda") if corpus == "g"
               else pink_frames(seed, W, H, args.frames))
        rf, tf = timed(an["full"], uhd, args.reps)
        rl, tl = timed(an["low"], uhd, args.reps)
        r2, _ = timed(an["1080"], downsample(uhd, 2), 1)
        r4, _ = timed(an["540"], downsample(uhd, 4), 1)
        row = {"corpus": corpus, "clip": ("G(%d)" if corpus == "g" else "pink(%d)") % seed, "frames": args.frames,
               "fps_full": args.frames / tf * 1e3, "fps_lowpass": args.frames / tl * 1e3, "speedup": tf / tl,
               "mean_E_Y": {"2160_full": float(rf["E_Y"].mean()), "2160_lowpass": float(rl["E_Y"].mean()),
                            "1080": float(r2["E_Y"].mean()), "540": float(r4["E_Y"].mean())},
               "pcc_frames_E_Y_low_vs_full": pcc(rf["E_Y"], rl["E_Y"]),
               "block": {"1080": an["1080"].info["block"][0], "540": an["540"].info["block"][0]}}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del uhd
        torch.cuda.empty_cache()
    m = {k: [r["mean_E_Y"][k] for r in rows] for k in rows[0]["mean_E_Y"]}
    summ = {"summary": True, "corpus": corpus, "clips": len(rows), "frames_per_clip": args.frames,
            "speedup_mean": float(np.mean([r["speedup"] for r in rows])),
            "speedup_min": float(np.min([r["speedup"] for r in rows])),
            "pcc_clip_mean_E_Y_lowpass_vs_full": pcc(m["2160_full"], m["2160_lowpass"]),
            "pcc_clip_mean_E_Y_2160_vs_1080": pcc(m["2160_full"], m["1080"]),
            "pcc_clip_mean_E_Y_2160_vs_540": pcc(m["2160_full"], m["540"]),
            "pcc_clip_mean_E_Y_1080_vs_540": pcc(m["1080"], m["540"]),
            "pcc_frames_E_Y_low_vs_full_min": float(np.nanmin([r["pcc_frames_E_Y_low_vs_full"] for r in rows])),
            "clip_mean_E_Y_2160_full_range": [float(min(m["2160_full"])), float(max(m["2160_full"]))]}
    summ["criteria"] = {"speedup_ge_1.8": summ["speedup_min"] >= 1.8,
                        "pcc_lowpass_ge_0.90": summ["pcc_clip_mean_E_Y_lowpass_vs_full"] >= 0.90,
                        "pcc_cross_res_ge_0.90": min(summ["pcc_clip_mean_E_Y_2160_vs_1080"],
                                                     summ["pcc_clip_mean_E_Y_2160_vs_540"],
                                                     summ["pcc_clip_mean_E_Y_1080_vs_540"]) >= 0.90}
    return rows, summ


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clips", type=int, default=24)
    ap.add_argument("--frames", type=int, default=48)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--first-seed", type=int, default=100)
    ap.add_argument("--corpus", default="both", choices=("g", "pink", "both"))
    ap.add_argument("--git", default=None, help="commit of the build (the GPU box has no .git)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    W, H = 3840, 2160
    an = {"full": Analyzer(W, H, 8, 32, False), "low": Analyzer(W, H, 8, 32, True),
          "1080": Analyzer(W // 2, H // 2, 8, 0, False), "540": Analyzer(W // 4, H // 4, 8, 0, False)}
    git = args.git
    if git is None:
        try:
            git = subprocess.run(["git", "rev-parse", "--short", "HEAD"], cwd=ROOT, capture_output=True,
                                 text=True).stdout.strip() or None
        except Exception:
            git = None
    t0 = time.time()
    allrows, summs = [], []
    for corpus in (("g", "pink") if args.corpus == "both" else (args.corpus,)):
        rows, summ = study(corpus, args, an)
        summ.update({"git": git, "gpu": torch.cuda.get_device_name(0), "elapsed_s": time.time() - t0})
        print(json.dumps(summ), flush=True)
        allrows += rows
        summs.append(summ)
    if args.out:
        with open(args.out, "w") as fh:
            for r in allrows:
                fh.write(json.dumps(r) + "\n")
            for sm in summs:
                fh.write(json.dumps(sm) + "\n")


if __name__ == "__main__":
    main()
