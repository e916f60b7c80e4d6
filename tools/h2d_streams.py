#!/usr/bin/env python
"""Pinned host->device copy bandwidth with 1, 2, 4 concurrent streams (is one copy engine the
PCIe limit?).  Prints GB/s per configuration."""
import torch

N = 1 << 30
host = torch.empty(N, dtype=torch.uint8, pin_memory=True)
host.fill_(1)
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = N // ns
    best = 0.0
    for rep in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dev[i * chunk:(i + 1) * chunk].copy_(host[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, N / (e0.elapsed_time(e1) / 1e3) / 1e9)
    print("streams %d: %.1f GB/s" % (ns, best))
# also chunked sequential 8 MB copies on one stream (like an 8-frame chunk pipeline)
for cb in (8 << 20, 64 << 20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(N // cb):
        dev[i * cb:(i + 1) * cb].copy_(host[i * cb:(i + 1) * cb], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print("one stream, %d MB chunks: %.1f GB/s" % (cb >> 20, N / (e0.elapsed_time(e1) / 1e3) / 1e9))
