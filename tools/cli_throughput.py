#!/usr/bin/env python
"""NEXT-3 measurement: end-to-end throughput of the file-based path (Y4M on local disk /
page cache -> native reader thread -> pinned batches -> PCIe -> kernels -> CSV) through the
native C client and the Python CLI, on synthetic UHD 8-bit frames (config 3 geometry)."""
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2304_12384_b200 import build, synth  # noqa: E402

F = int(os.environ.get("CLI_FRAMES", "120"))
W, H = 3840, 2160
tmp = tempfile.mkdtemp(prefix="vca_cli_")
path = os.path.join(tmp, "clip.y4m")
Y, U, V = synth.config_frames(3, device="cuda", n_frames=F)
Y, U, V = (p.cpu().numpy() for p in (Y, U, V))
with open(path, "wb") as fh:
    fh.write(b"YUV4MPEG2 W%d H%d F50:1 Ip A1:1 C420jpeg\n" % (W, H))
    for t in range(F):
        fh.write(b"FRAME\n")
        fh.write(Y[t].tobytes())
        fh.write(U[t].tobytes())
        fh.write(V[t].tobytes())
size = os.path.getsize(path)
res = {"frames": F, "file_bytes": size}
for name, cmd in (("native_vca_cli", [build.CLI, path, "-o", os.path.join(tmp, "c.csv"), "--block", "32", "--low-pass"]),
                  ("python_cli", [sys.executable, "-m", "paper_2304_12384_b200.cli", "analyze", path, "-o",
                                  os.path.join(tmp, "p.csv"), "--block-size", "32", "--low-pass"])):
    subprocess.run(cmd, cwd=ROOT, capture_output=True)  # warm the page cache / CUDA context
    t0 = time.perf_counter()
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    wall = time.perf_counter() - t0
    line = [l for l in r.stderr.splitlines() if l.startswith("# frames=")]
    res[name] = {"rc": r.returncode, "wall_s_incl_startup": wall, "reported": line[0] if line else r.stderr[-300:]}
same = open(os.path.join(tmp, "c.csv"), "rb").read() == open(os.path.join(tmp, "p.csv"), "rb").read()
res["csv_identical"] = same
print(json.dumps(res))
