#!/usr/bin/env python
"""Probe: can a read-only mmap of a (page-cached) frame file be page-locked with
cudaHostRegister, and how fast is registration and the H2D copy from it?  (Zero-copy ingest
would skip the pread memcpy into pinned staging.)"""
import ctypes
import glob
import mmap
import os
import time

import numpy as np
import torch

fn = "/tmp/regtest.bin"
size = 1_492_992_000  # 120 UHD 8-bit frames
if not os.path.exists(fn) or os.path.getsize(fn) != size:
    with open(fn, "wb") as f:
        chunk = os.urandom(1 << 20) * 64
        left = size
        while left > 0:
            n = min(left, len(chunk))
            f.write(chunk[:n])
            left -= n
lib = ctypes.CDLL((glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*"))
                   + glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
torch.zeros(1, device="cuda")
dev = torch.empty(size, dtype=torch.uint8, device="cuda")
for label, flags in (("readonly-flag", 0x08), ("default", 0x00), ("portable", 0x01), ("mapped", 0x02)):
    fd = os.open(fn, os.O_RDONLY)
    mm = mmap.mmap(fd, size, prot=mmap.PROT_READ)
    a = np.frombuffer(mm, dtype=np.uint8)
    ptr = a.ctypes.data
    a[::4096].sum()  # fault the pages in
    t0 = time.perf_counter()
    rc = lib.cudaHostRegister(ctypes.c_void_p(ptr), ctypes.c_size_t(size), ctypes.c_uint(flags))
    t1 = time.perf_counter()
    lib.cudaGetLastError()
    msg = "%-14s register rc %d in %.1f ms" % (label, rc, (t1 - t0) * 1e3)
    if rc == 0:
        src = torch.from_numpy(a)
        best = 0
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, size / (time.perf_counter() - t0) / 1e9)
        msg += ", H2D %.1f GB/s" % best
        lib.cudaHostUnregister(ctypes.c_void_p(ptr))
    print(msg, flush=True)
    del a
    mm.close()
    os.close(fd)
os.remove(fn)
