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
buf = (ctypes.c_ulonglong * (3 * groups))()
for rep in range(4):
    a.reset(0)
    a.analyze(Y, U, V)
    torch.cuda.synchronize()
    assert L.vca_debug_group_times(buf, groups) == 0
    raw = np.frombuffer(buf, dtype=np.uint64).reshape(3, groups)
    t = raw[:2].astype(np.float64)
    smid = raw[2].astype(np.int64)
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
    if rep == 3:
        grp = np.arange(groups) % 3
        for g in range(3):
            print("  group slot %d: us/item median %.3f" % (g, np.median(rate[grp == g])))
        # per SM: mean rate of its groups; SMs in id order (TPC pairs, GPCs)
        sm_rate = {}
        for v in range(groups):
            sm_rate.setdefault(int(smid[v]), []).append(rate[v])
        ids = sorted(sm_rate)
        r = np.array([np.mean(sm_rate[i]) for i in ids])
        print("  SMs %d; per-SM us/item min %.3f median %.3f max %.3f; lower/upper half of SM ids %.3f / %.3f"
              % (len(ids), r.min(), np.median(r), r.max(), r[: len(r) // 2].mean(), r[len(r) // 2:].mean()))
        slow = [ids[i] for i in np.argsort(r)[-10:]]
        fast = [ids[i] for i in np.argsort(r)[:10]]
        print("  slowest SM ids", sorted(slow), " fastest", sorted(fast))
        print("  rate spread within an SM (max - min over its 3 groups), median %.3f us/item"
              % np.median([max(v) - min(v) for v in sm_rate.values()]))
