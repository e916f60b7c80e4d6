#!/usr/bin/env python
"""Diagnostic: per-consumer-group start / end times of the fused block kernel (a VCA_TIMES build,
selected with VCA_LIB), to size the static schedule's tail.  usage: VCA_LIB=... group_times.py [cfg]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_12384_b200 import Analyzer, synth, vca  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = synth.CONFIGS[cfg]
Y, U, V = synth.config_frames(cfg, device="cuda")
a = Analyzer(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
L = vca.lib()
groups = torch.cuda.get_device_properties(0).multi_processor_count * 3
buf = (ctypes.c_ulonglong * (2 * groups))()
for rep in range(4):
    a.reset(0)
    a.analyze(Y, U, V)
    torch.cuda.synchronize()
    assert L.vca_debug_group_times(buf, groups) == 0
    t = np.frombuffer(buf, dtype=np.uint64).astype(np.float64).reshape(2, groups)
    t0 = t[0].min()
    st, en = (t[0] - t0) / 1e3, (t[1] - t0) / 1e3
    items = c.n_frames * a.info["rows"][0]
    per = np.array([len(range(g, items, groups)) for g in range(groups)])
    rate = (en - st) / per
    print("cfg %d rep %d: start max %.1f us; end min %.1f median %.1f max %.1f us; us/item median %.2f "
          "(p5 %.2f, p95 %.2f); groups with %d items end median %.1f, with %d items %.1f"
          % (cfg, rep, st.max(), en.min(), np.median(en), en.max(), np.median(rate), np.percentile(rate, 5),
             np.percentile(rate, 95), per.max(), np.median(en[per == per.max()]), per.min(),
             np.median(en[per == per.min()])))
