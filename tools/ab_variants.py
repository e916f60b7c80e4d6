#!/usr/bin/env python
"""A/B timing of libvca build variants (paper_2304_12384_b200/variants/*.so) on
one workload, frames generated once.  Prints fps per variant and checks that
every variant's records equal the first variant's bit for bit."""
import glob
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_12384_b200 import synth, vca  # noqa: E402


def main():
    """Parent: run every variant in its own process under a timeout (a hung kernel
    must not hang the whole call).  Child (--one PATH): time one variant."""
    if "--one" not in sys.argv:
        import subprocess
        libs = sys.argv[1:] or sorted(glob.glob(os.path.join(ROOT, "paper_2304_12384_b200", "variants", "*.so")))
        results = {}
        for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
            for path in libs:
                try:
                    r = subprocess.run([sys.executable, __file__, "--one", path, str(rnd)], capture_output=True,
                                       text=True, timeout=int(os.environ.get("AB_TIMEOUT", "120")))
                    sys.stdout.write(r.stdout + (r.stderr[-2000:] if r.returncode else ""))
                    for line in r.stdout.splitlines():
                        if " fps " in line:
                            results.setdefault(os.path.basename(path), []).append(float(line.split()[5]))
                except subprocess.TimeoutExpired:
                    print("round %d %-28s TIMEOUT" % (rnd, os.path.basename(path)))
                sys.stdout.flush()
        for name, v in results.items():
            print("median %-28s %9.0f fps over %d rounds" % (name, sorted(v)[len(v) // 2], len(v)))
        return
    one(sys.argv[sys.argv.index("--one") + 1], int(sys.argv[-1]))


def one(path, rnd):
    cfg = int(os.environ.get("AB_CONFIG", "3"))
    frames = int(os.environ.get("AB_FRAMES", "600"))
    steps = int(os.environ.get("AB_STEPS", "20"))
    c = synth.CONFIGS[cfg]
    Y, U, V = synth.config_frames(cfg, device="cuda", n_frames=frames)
    fb = (c.width * c.height + 2 * (c.width // 2) * (c.height // 2)) * (1 if c.bit_depth == 8 else 2)
    ref = None
    for _ in (0,):
        for path in (path,):
            vca._lib = None
            os.environ["VCA_LIB"] = path
            a = vca.Analyzer(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
            out = torch.empty((frames, 8), dtype=torch.float64, device="cuda")
            for _ in range(3):
                a.reset(0)
                a.analyze(Y, U, V, out=out)
            torch.cuda.synchronize()
            a.profile_read()
            a.profile_enable(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                a.reset(0)
                a.analyze(Y, U, V, out=out)
            e1.record()
            torch.cuda.synchronize()
            blk, fin, n = a.profile_read()
            ms = e0.elapsed_time(e1) / steps
            rec = vca.records_to_numpy(out)
            refp = os.path.join(ROOT, "gpurun_out", "ab_ref_%d_%d.npy" % (cfg, frames))
            if not os.path.exists(refp):
                np.save(refp, rec)
                same = "(reference)"
            else:
                ref = np.load(refp)
                same = "identical" if np.array_equal(rec, ref) else (
                    "maxrel %.3g" % max(float(np.max(np.abs(rec[f] - ref[f]) / np.maximum(np.abs(ref[f]), 1e-300)))
                                        for f in vca.FEATURES))
            print("round %d %-28s %8.3f ms/step  %9.0f fps  kernel %.3f ms (%.0f GB/s)  %s" % (
                rnd, os.path.basename(path), ms, frames / ms * 1e3, blk / steps, frames * fb / (blk / steps) / 1e6,
                same), flush=True)
            a.close()


if __name__ == "__main__":
    main()
