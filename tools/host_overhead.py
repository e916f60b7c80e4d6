import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2304_12384_b200 import Analyzer, synth
for cfg in (1, 3):
    c = synth.CONFIGS[cfg]
    F = c.n_frames if cfg == 1 else 60
    Y, U, V = synth.with_pitch(synth.config_frames(cfg, device="cuda", n_frames=F))
    a = Analyzer(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
    out = torch.empty((F, 8), dtype=torch.float64, device="cuda")
    scratch = torch.empty(a.scratch_bytes(F) // 8 + 1, dtype=torch.float64, device="cuda")
    for _ in range(5): a.analyze(Y, U, V, out=out, scratch=scratch)
    torch.cuda.synchronize()
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(n): a.analyze(Y, U, V, out=out, scratch=scratch)
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    gpu = e0.elapsed_time(e1) / n * 1e3
    host = (t1 - t0) / n * 1e6
    print("config %d: %.1f us per call on the GPU stream, %.1f us host enqueue per call" % (cfg, gpu, host))

# the C call alone (arguments marshalled once): what the library itself costs per call
from paper_2304_12384_b200.vca import _plane_args  # noqa: E402

c = synth.CONFIGS[1]
Y, U, V = synth.with_pitch(synth.config_frames(1, device="cuda", n_frames=16))
a = Analyzer(c.width, c.height, 8, 32, False)
out = torch.empty((16, 8), dtype=torch.float64, device="cuda")
scratch = torch.empty(a.scratch_bytes(16) // 8 + 1, dtype=torch.float64, device="cuda")
ptrs, pitch, fstride = _plane_args((Y, U, V), True)
st = torch.cuda.current_stream().cuda_stream
args = (a._h, ptrs, pitch, fstride, 16, 0, scratch.data_ptr(), scratch.numel() * 8, out.data_ptr(), st)
for _ in range(5):
    a._L.vca_analyze(*args)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    a._L.vca_analyze(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("config 1: %.1f us per vca_analyze C call (host)" % ((t1 - t0) / 200 * 1e6))
