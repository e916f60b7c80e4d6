#!/usr/bin/env python
"""Largest relative difference per feature between the CUDA path and the oracle (first 120
frames of configs 1-4): how far inside the 1e-6 parity bar the FP64 epilogue sits."""
import sys, numpy as np, torch
import os; _R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, _R)
import oracle
from paper_2304_12384_b200 import Analyzer, records_to_numpy, synth
FEATS = ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V")
for cfg in (2, 3, 4, 1):
    c = synth.CONFIGS[cfg]
    F = min(c.n_frames, 120)
    Y, U, V = synth.config_frames(cfg, device="cuda", n_frames=F)
    if cfg == 1:
        Y, U, V = synth.with_pitch((Y, U, V))
    a = Analyzer(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
    g = records_to_numpy(a.analyze(Y, U, V))
    r = oracle.analyze(*synth.as_numpy_planes(Y, U, V), c.bit_depth, c.block_size, c.lowpass)
    out = []
    for f in FEATS:
        nz = r[f] != 0
        rel = np.abs(g[f][nz] - r[f][nz]) / np.abs(r[f][nz])
        out.append("%s %.2e" % (f, rel.max() if rel.size else 0.0))
    print(cfg, "  ".join(out), flush=True)
