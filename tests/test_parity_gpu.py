"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded bytes.  Bar (BASELINE.json north star; R-11): integer DCT
coefficients, DC sums and per-block AC checksums bit-exact; per-frame features
within 1e-6 relative, an exact 0 reproduced as exactly 0; the production kernel
instantiation bit-identical to the DUMP instantiation that exposes the integers
(see tests/parity_util.py)."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2304_12384_b200 import Analyzer, records_to_numpy, synth
from parity_util import FEATS, RTOL, Pair, assert_checks, assert_records, oracle_checks, planes_cuda  # noqa: F401

pytestmark = pytest.mark.gpu


def run_both(Y, U, V, bd, w, lp, n_halo=0):
    """Y, U, V torch CPU tensors -> (gpu records, oracle records)."""
    a = Analyzer(Y.shape[2], Y.shape[1], bd, w, lp)
    rec = a.analyze(*planes_cuda(Y, U, V), n_halo=n_halo)
    torch.cuda.synchronize()
    g = records_to_numpy(rec)
    r = oracle.analyze(*synth.as_numpy_planes(Y, U, V), bd, w, lp, n_halo=n_halo)
    return g, r, a


def check_dump(a, Y, U, V, bd, w, lp, frame=0):
    """Bit-exact coefficients / DC sums / per-block H, L of one frame."""
    dump = a.debug_dump(*planes_cuda(Y[frame:frame + 1], U[frame:frame + 1], V[frame:frame + 1]))
    npl = synth.as_numpy_planes(Y[frame:frame + 1], U[frame:frame + 1], V[frame:frame + 1])
    info = a.info
    for p in range(3):
        plane = npl[p][0]
        wp, n = info["block"][p], info["n"][p]
        k = 0
        for r in range(info["rows"][p]):
            for c in range(info["cols"][p]):
                C, sumx, H, L = oracle.block(plane, bd, wp, lp, r, c)
                got = dump[p]["coeffs"][k].astype(np.int64)
                want = C.copy()
                want[0, 0] = np.int64(np.uint32(want[0, 0] & 0xFFFFFFFF).view(np.int32))  # C_00 mod 2^32 (R-11)
                assert np.array_equal(got, want), (p, r, c)
                assert dump[p]["sumx"][k] == sumx and 4096 * sumx == C[0, 0]
                assert dump[p]["L"][k] == L                      # same correctly-rounded sqrt
                assert abs(dump[p]["H"][k] - H) <= 1e-12 * max(H, 1e-300)
                k += 1


CASES = [
    # (name, W, H, bit depth, block, lowpass)  -- small geometries spanning several tiles + ragged tails
    ("cif_full32", 352, 288, 8, 32, False),           # config 1 geometry
    ("ragged_full32", 200, 136, 8, 32, False),        # config 2 family: partial last row AND column
    ("ragged_lp32", 264, 176, 8, 32, True),           # config 3 family: last row 16/32
    ("ragged_10bit_full16", 136, 100, 10, 16, False),  # config 4 family
    ("lp32_10bit", 128, 96, 10, 32, True),
    ("full16_8bit", 160, 88, 8, 16, False),
    ("lp16", 96, 72, 8, 16, True),                     # generic kernel: n = 8 / 4
    ("full8", 72, 46, 8, 8, False),
    ("full4", 38, 22, 8, 4, False),                    # chroma grid differs from luma grid
    ("full4_10bit", 40, 24, 10, 4, False),
    ("tiny_8x8", 8, 8, 8, 32, False),                  # plane smaller than a block
]


# Several whole strips of the fused kernel (16 units per strip for n = 16 luma, 8 for
# n = 32 and for the 10-bit low-pass family) plus a ragged strip end, a partial last block
# column inside a strip and a partial last block row.
CASES_STRIPS = [
    ("strips_lp32", 1174, 100, 8, 32, True),          # 37 cols: 2 x 16 + 5, last col 22/32 wide
    ("strips_full16_10bit", 586, 72, 10, 16, False),   # 37 cols, last col 10/16 wide
    ("strips_full32", 602, 76, 8, 32, False),          # 19 cols: 2 x 8 + 3, last col 26/32 wide
    ("strips_lp32_10bit", 602, 68, 10, 32, True),      # 19 cols (8-unit strips)
    ("strips_full16_8bit", 1040, 40, 8, 16, False),    # 65 cols: 4 x 16 + 1
    # n = 8 luma / n = 4 chroma families (luma pairs + 8-block chroma MMA per warp)
    ("strips_lp16", 586, 70, 8, 16, True),             # 37 cols: 2 x 16 + 5, last col 10/16, last row 6/16
    ("strips_lp16_10bit", 586, 40, 10, 16, True),
    ("strips_full8", 294, 30, 8, 8, False),            # 37 cols, last col 6/8 wide, last row 6/8
    ("strips_full8_10bit", 294, 22, 10, 8, False),
    # w = 4 (thread-per-block kernel; chroma grid half the luma grid)
    ("wide_full4", 602, 70, 8, 4, False),
    ("wide_full4_10bit", 330, 38, 10, 4, False),
    # row bytes a multiple of the box width: the 4-D tensor-map loads (one TMA per plane per
    # strip); partial last block row, ragged last strip
    ("tma4_lp16", 1152, 70, 8, 16, True),              # 72 cols: 4 x 16 + 8; Y 4-D, chroma 3-D
    ("tma4_full16_8bit", 1152, 40, 8, 16, False),      # Y 4-D, chroma 3-D (one box per strip)
    ("tma4_full16_10bit", 640, 40, 10, 16, False),     # 40 cols: 2 x 16 + 8; Y and chroma 4-D
    ("tma4_lp32_10bit", 1024, 68, 10, 32, True),
    ("tma4_full32", 1280, 76, 8, 32, False),           # 40 cols: 5 x 8; Y 4-D, chroma 3-D (640 B rows)
]


@pytest.mark.parametrize("name,W,H,bd,w,lp", CASES + CASES_STRIPS, ids=[c[0] for c in CASES + CASES_STRIPS])
def test_parity_small(name, W, H, bd, w, lp):
    """Records against the oracle, the production instantiation against the DUMP one bit for
    bit, every block's integer checks of every frame, every coefficient of frame 1."""
    F = 4
    Y, U, V = synth.g_frames(17, W, H, F, bd)
    g, r, a = run_both(Y, U, V, bd, w, lp)
    assert_records(g, r)
    pair = Pair(W, H, bd, w, lp)
    rec, hy, ch = pair.analyze(*planes_cuda(Y, U, V))
    ro, rhy, rch = oracle_checks(Y, U, V, bd, w, lp)
    assert rec.tobytes() == g.tobytes()
    assert_records(rec, ro, rtol=1e-12)
    assert_checks(ch, rch)
    check_dump(a, Y, U, V, bd, w, lp, frame=1)


def test_parity_config1_cif_all_frames():
    """Config 1 whole (16 CIF frames, one call): records at 1e-6 and 1e-12, every block's H_Y,
    production == DUMP instantiation bit for bit, every block's integer checks, and every
    coefficient of every frame (SURVEY 8(c) "Whole pipeline")."""
    Y, U, V = synth.config_frames(1)
    pair = Pair(352, 288, 8, 32, False)
    g, HY, ch = pair.analyze(*planes_cuda(Y, U, V))
    r, rHY, rch = oracle_checks(Y, U, V, 8, 32, False)
    assert_records(g, r)
    assert_records(g, r, rtol=1e-12)
    assert np.all(np.abs(HY - rHY) <= 1e-12 * np.maximum(rHY, 1e-300))
    assert_checks(ch, rch)
    for t in range(16):
        check_dump(pair.prod, Y, U, V, 8, 32, False, frame=t)


def test_extreme_values():
    """Saturated / zero / checkerboard frames: exact zeros, int32 headroom at 10-bit (R-11)."""
    for bd, w, lp in ((8, 32, False), (10, 16, False), (8, 32, True), (10, 32, True), (10, 8, False)):
        hi = (1 << bd) - 1
        dt = torch.uint8 if bd == 8 else torch.int16
        W, H = 96, 64
        yy, xx = torch.meshgrid(torch.arange(H), torch.arange(W), indexing="ij")
        cb = ((xx + yy) % 2) * hi
        frames = [torch.zeros(H, W), torch.full((H, W), float(hi)), cb.float(), torch.zeros(H, W)]
        Y = torch.stack(frames).to(dt)
        U = torch.stack([f[: H // 2, : W // 2] for f in frames]).to(dt)
        V = torch.stack([f[: H // 2, : W // 2].flip(1) for f in frames]).to(dt)
        g, r, a = run_both(Y, U, V, bd, w, lp)
        assert_records(g, r)
        assert g["E_Y"][0] == 0.0 and g["h"][1] == 0.0 and g["L_Y"][0] == 0.0
        check_dump(a, Y, U, V, bd, w, lp, frame=2)


def test_ten_bit_clamp_gpu():
    """container values > 1023 are clamped (kernel and oracle alike)."""
    Y, U, V = synth.g_frames(3, 64, 48, 2, 10)
    Y[0, 5, 7] = 4000
    U[1, 3, 3] = 2000
    g, r, _ = run_both(Y, U, V, 10, 16, False)
    assert_records(g, r)


def test_split_and_halo_invariance():
    """S:362/S:379 analog: any chunking of the sequence into calls (carried
    H_Y) or a range split with a one-frame halo is bit-identical."""
    Y, U, V = planes_cuda(*synth.g_frames(23, 264, 176, 9, 8))  # 264: pitch 272 (padded)
    a = Analyzer(264, 176, 8, 32, True)
    whole = records_to_numpy(a.analyze(Y, U, V))
    b = Analyzer(264, 176, 8, 32, True)
    parts = []
    for s, e in ((0, 2), (2, 3), (3, 9)):
        parts.append(records_to_numpy(b.analyze(Y[s:e], U[s:e], V[s:e])))
    assert np.array_equal(np.concatenate(parts), whole)
    # two "ranks": [0, 5) and [5, 9) with halo frame 4
    c = Analyzer(264, 176, 8, 32, True)
    c.reset(5)
    tail = records_to_numpy(c.analyze(Y[4:], U[4:], V[4:], n_halo=1))
    assert np.array_equal(tail, whole[5:])
    # reset starts a new sequence: h = 0
    b.reset(0)
    again = records_to_numpy(b.analyze(Y[3:5], U[3:5], V[3:5]))
    assert again["h"][0] == 0.0 and again["poc"][0] == 0


def test_analyze_host_matches_device():
    Yc, Uc, Vc = synth.with_pitch(synth.g_frames(31, 200, 136, 7, 8))
    Yp, Up, Vp = (torch.empty_strided(p.shape, p.stride(), dtype=p.dtype, pin_memory=True) for p in (Yc, Uc, Vc))
    for d, s_ in zip((Yp, Up, Vp), (Yc, Uc, Vc)):
        d.copy_(s_)
    a = Analyzer(200, 136, 8, 32, False)
    dev = records_to_numpy(a.analyze(*planes_cuda(Yc, Uc, Vc)))
    b = Analyzer(200, 136, 8, 32, False)
    host = b.analyze_host(Yp, Up, Vp, chunk_frames=3)
    assert np.array_equal(host, dev)
    c = Analyzer(200, 136, 8, 32, False)
    c.reset(1)
    host2 = c.analyze_host(Yc, Uc, Vc, n_halo=1, chunk_frames=2)  # pageable memory, halo frame 0
    assert np.array_equal(host2, dev[1:])


def test_analyze_host_error_leaves_sequence_unchanged():
    """vca.h: an argument error leaves the context unchanged -- a failed vca_analyze_host between
    two good calls does not advance the POC or the carried H_Y (records equal one uninterrupted
    sequence bit for bit)."""
    from paper_2304_12384_b200 import VcaError

    Yc, Uc, Vc = synth.with_pitch(synth.g_frames(33, 200, 136, 6, 8))
    whole = records_to_numpy(Analyzer(200, 136, 8, 32, False).analyze(*planes_cuda(Yc, Uc, Vc)))
    a = Analyzer(200, 136, 8, 32, False)
    first = a.analyze_host(Yc[:3], Uc[:3], Vc[:3], chunk_frames=2)
    with pytest.raises(VcaError) as e:
        a.analyze_host(Yc[3:4], Uc[3:4], Vc[3:4], n_halo=1)  # n_frames < 1 + n_halo
    assert e.value.code == -1
    rest = a.analyze_host(Yc[3:], Uc[3:], Vc[3:], chunk_frames=2)
    assert np.array_equal(np.concatenate([first, rest]), whole)


def test_contexts_on_concurrent_streams():
    """vca.h: one context per stream -- two contexts of different families (8-bit low-pass 32,
    10-bit full 16) launched alternately on two streams, several calls each, give the records of
    the same calls made one after another on one stream, bit for bit (no state shared between
    contexts: occupancy caches, tensor maps, scratch, carried H_Y)."""
    Ya, Ua, Va = planes_cuda(*synth.g_frames(41, 264, 200, 6, 8))
    Yb, Ub, Vb = planes_cuda(*synth.g_frames(42, 176, 112, 6, 10))
    ref_a = Analyzer(264, 200, 8, 32, True)
    ref_b = Analyzer(176, 112, 10, 16, False)
    want_a = [records_to_numpy(ref_a.analyze(Ya[k:k + 2], Ua[k:k + 2], Va[k:k + 2])) for k in (0, 2, 4)]
    want_b = [records_to_numpy(ref_b.analyze(Yb[k:k + 2], Ub[k:k + 2], Vb[k:k + 2])) for k in (0, 2, 4)]
    a = Analyzer(264, 200, 8, 32, True)
    b = Analyzer(176, 112, 10, 16, False)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs_a = [torch.empty((2, 8), dtype=torch.float64, device="cuda") for _ in range(3)]
    outs_b = [torch.empty((2, 8), dtype=torch.float64, device="cuda") for _ in range(3)]
    scr_a = torch.empty(a.scratch_bytes(2) // 8 + 1, dtype=torch.float64, device="cuda")
    scr_b = torch.empty(b.scratch_bytes(2) // 8 + 1, dtype=torch.float64, device="cuda")
    for i, k in enumerate((0, 2, 4)):
        a.analyze(Ya[k:k + 2], Ua[k:k + 2], Va[k:k + 2], out=outs_a[i], scratch=scr_a, stream=s1)
        b.analyze(Yb[k:k + 2], Ub[k:k + 2], Vb[k:k + 2], out=outs_b[i], scratch=scr_b, stream=s2)
    torch.cuda.synchronize()
    for i in range(3):
        assert np.array_equal(records_to_numpy(outs_a[i]), want_a[i])
        assert np.array_equal(records_to_numpy(outs_b[i]), want_b[i])


def test_argument_errors_gpu():
    from paper_2304_12384_b200 import VcaError

    a = Analyzer(64, 64, 8, 32, False)
    Y = torch.zeros((2, 64, 64), dtype=torch.uint8, device="cuda")
    U = torch.zeros((2, 32, 32), dtype=torch.uint8, device="cuda")
    Ywide = torch.zeros((2, 64, 80), dtype=torch.uint8, device="cuda")
    with pytest.raises(VcaError) as e:
        a.analyze(Ywide[:, :, 1:65], U, U)     # large enough, but the base is not 16-byte aligned
    assert e.value.code == -6
    with pytest.raises(ValueError):
        a.analyze(Y[:, :, 1:], U, U)           # smaller than the context's plane: refused by the binding
    with pytest.raises(ValueError):
        a.analyze(Y, U, U, out=torch.empty((1, 8), dtype=torch.float64, device="cuda"))  # records buffer too small
    with pytest.raises(VcaError) as e:
        a.analyze(Y[:1], U[:1], U[:1], n_halo=1)  # n_frames < 1 + n_halo
    assert e.value.code == -1
    small = torch.empty(1, dtype=torch.float64, device="cuda")
    with pytest.raises(VcaError) as e:
        a.analyze(Y, U, U, scratch=small)
    assert e.value.code == -9
    # the context is still usable after argument errors
    rec = records_to_numpy(a.analyze(Y, U, U))
    assert np.all(rec["E_Y"] == 0.0)


def test_profile_counters():
    a = Analyzer(128, 64, 8, 32, True)
    Y, U, V = planes_cuda(*synth.g_frames(1, 128, 64, 3, 8))
    a.profile_enable(True)
    a.analyze(Y, U, V)
    a.analyze(Y, U, V)
    blk, fin, launches = a.profile_read()
    assert blk > 0 and fin > 0 and launches == 4


@pytest.mark.slow
@pytest.mark.parametrize("cfg", (2, 3, 4))
def test_parity_full_size_all_frames(cfg):
    """Full BASELINE.json geometry and batch, analysed in one call (the launch configuration
    bench.py times): the production instantiation bit-identical to the DUMP instantiation
    (records and every block's H_Y), and against the oracle every record, every block's H_Y and
    the exact integer checks (AC checksum, sample sum) of every block of every plane of every
    frame (chunks behind a one-frame halo for h), every feature finite and non-negative, and
    the coefficient dump of the last frame."""
    c = synth.CONFIGS[cfg]
    F = c.n_frames            # the whole BASELINE.json batch in one call, as bench.py times it
    Y, U, V = synth.config_frames(cfg, device="cuda", n_frames=F)
    pair = Pair(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
    g, HY, ch = pair.analyze(Y, U, V)
    assert len(g) == F and np.array_equal(g["poc"], np.arange(F))
    for f in FEATS:            # properties of every frame: finite, non-negative
        assert np.all(np.isfinite(g[f])) and np.all(g[f] >= 0.0), f
    step = 40
    for s in range(0, F, step):
        e = min(F, s + step)
        h0 = 1 if s > 0 else 0
        r, rHY, rch = oracle_checks(Y[s - h0:e], U[s - h0:e], V[s - h0:e], c.bit_depth, c.block_size, c.lowpass,
                                    n_halo=h0, first_poc=s)
        assert_records(g[s:e], r)
        # the sides differ only in FP64 summation order (<= 2e-14 measured,
        # tests/test_parity_margins_gpu.py), so 1e-12 also holds.  It does NOT pin single
        # chroma coefficients: one wrong config-4 chroma coefficient moves E_U or E_V by only
        # ~3e-13..8e-13 relative (w / (4096 n) / (C n^2) against E ~ 50); the per-block
        # integer checks below are what pin every coefficient.
        assert_records(g[s:e], r, rtol=1e-12)
        want = rHY[h0:]
        assert np.all(np.abs(HY[s:e] - want) <= 1e-12 * np.maximum(want, 1e-300)), s
        assert_checks(ch, [{k: v[h0:] for k, v in d.items()} for d in rch], frames=slice(s, e))
    Yc, Uc, Vc = (p[F - 1:F].cpu() for p in (Y, U, V))
    check_dump(pair.prod, Yc, Uc, Vc, c.bit_depth, c.block_size, c.lowpass, frame=0)


@pytest.mark.slow
def test_parity_config5_all_frames():
    """Config 5 whole: 4800 UHD frames (8 segments G(10..17)) analysed as one sequence, segment
    by segment on one context pair (the carried H_Y crosses every segment cut), production ==
    DUMP bit for bit, every record, H_Y and per-block integer check of every frame against the
    oracle (which gets the previous segment's H_Y as prev_HY), and GPU-count invariance: at each
    of the 7 segment boundaries -- every rank start of the 2-, 4- and 8-GPU splits
    (shard.plan) -- a fresh context behind a one-frame halo gives the same records bit for bit."""
    from paper_2304_12384_b200 import shard

    c = synth.CONFIGS[5]
    S = synth.SEGMENT_FRAMES
    starts = sorted({shard.plan(c.n_frames, wd, r).first_poc for wd in (2, 4, 8) for r in range(wd)} - {0})
    assert starts == [S * k for k in range(1, 8)]
    pair = Pair(c.width, c.height, 8, c.block_size, c.lowpass)
    prev_HY = None
    prev_last = None
    for seg in range(c.n_frames // S):
        Y, U, V = synth.config_frames(5, device="cuda", n_frames=S, first_t=seg * S)
        g, HY, ch = pair.analyze(Y, U, V)
        assert np.array_equal(g["poc"], np.arange(seg * S, (seg + 1) * S))
        step = 60
        for s in range(0, S, step):
            e = min(S, s + step)
            prev = prev_HY if s == 0 else HY[s - 1]
            r, rHY, rch = oracle_checks(Y[s:e], U[s:e], V[s:e], 8, c.block_size, c.lowpass, first_poc=seg * S + s,
                                        prev_HY=prev)
            assert_records(g[s:e], r)
            assert_records(g[s:e], r, rtol=1e-12)
            assert np.all(np.abs(HY[s:e] - rHY) <= 1e-12 * np.maximum(rHY, 1e-300)), (seg, s)
            assert_checks(ch, rch, frames=slice(s, e))
        if seg > 0:
            # a rank starting at this segment: fresh context, halo = the previous segment's last frame
            assert g["h"][0] > 0.0            # h across the cut, not a sequence restart
            b = Analyzer(c.width, c.height, 8, c.block_size, c.lowpass)
            b.reset(seg * S)
            Yh, Uh, Vh = (torch.cat([q, p]) for q, p in zip(prev_last, (Y, U, V)))
            ranked = records_to_numpy(b.analyze(Yh, Uh, Vh, n_halo=1))
            assert ranked.tobytes() == g.tobytes(), seg
            del Yh, Uh, Vh, b
        prev_HY = HY[-1].copy()
        prev_last = tuple(p[-1:].clone() for p in (Y, U, V))
        del Y, U, V
        torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("world", (2, 4, 8))
def test_config5_rank_boundary_full_size(world):
    """Config 5 at full UHD size: the rank that starts at a segment boundary (shard.plan) analyses
    its first frames behind a one-frame halo taken from the previous segment; its records equal a
    single call across the boundary bit for bit (GPU-count invariance) and the oracle."""
    from paper_2304_12384_b200 import shard

    c = synth.CONFIGS[5]
    sh = shard.plan(c.n_frames, world, 1)
    k = 4                                             # records checked after the boundary
    Y, U, V = synth.config_frames(5, device="cuda", n_frames=k + 2, first_t=sh.first_poc - 2)
    a = Analyzer(c.width, c.height, 8, c.block_size, c.lowpass)
    a.reset(sh.first_poc - 2)
    whole = records_to_numpy(a.analyze(Y, U, V))
    b = Analyzer(c.width, c.height, 8, c.block_size, c.lowpass)
    b.reset(sh.first_poc)
    ranked = records_to_numpy(b.analyze(Y[1:], U[1:], V[1:], n_halo=sh.n_halo))
    assert ranked["poc"][0] == sh.first_poc and ranked.tobytes() == whole[2:].tobytes()
    npl = synth.as_numpy_planes(Y[1:3].cpu(), U[1:3].cpu(), V[1:3].cpu())
    r = oracle.analyze(*npl, 8, c.block_size, c.lowpass, n_halo=1, first_poc=sh.first_poc)
    assert_records(ranked[:1], r)
    assert ranked["h"][0] > 0.0                       # h across the segment cut, not a restart


@pytest.mark.slow
def test_parity_8k_two_frames():
    """Largest geometry in use (8K UHD-2, 7680x4320, block 32 low-pass and full): all seven
    features of both frames (h across them) against the oracle."""
    Y, U, V = synth.g_frames(21, 7680, 4320, 2, 8)
    for lp in (True, False):
        g, r, a = run_both(Y, U, V, 8, 32, lp)
        assert_records(g, r)


@pytest.mark.parametrize("mode", ("full", "lowpass"))
def test_golden_closed_form_gpu(mode):
    """tests/golden/derived.json (closed form from the definitions) through the
    CUDA path: E_Y = w* a / n, h = w* |a1 - a0| / n, L = sqrt(v n)."""
    import json
    import os

    from test_oracle_pins import _fixture_frames

    g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                    "derived.json")))["closed_form_frames"][mode]
    Y, U, V = (torch.from_numpy(p) for p in _fixture_frames((50, 20), mode == "lowpass"))
    a = Analyzer(Y.shape[2], Y.shape[1], 8, 32, mode == "lowpass")
    rec = records_to_numpy(a.analyze(*planes_cuda(Y, U, V)))
    assert rec["E_Y"].tolist() == pytest.approx(g["E_Y"], rel=1e-14)
    assert rec["h"][0] == 0.0 and rec["h"][1] == pytest.approx(g["h"][1], rel=1e-14)
    for f in ("L_Y", "L_U", "L_V"):
        assert rec[f].tolist() == pytest.approx([g[f]] * 2, rel=1e-15)
    assert np.all(rec["E_U"] == 0.0) and np.all(rec["E_V"] == 0.0)


@pytest.mark.parametrize("W,H,bd,w,lp", [
    (2, 2, 8, 32, False),        # smallest accepted frame (R-12): one partial block per plane
    (2, 2, 10, 8, False),
    (16384, 34, 8, 32, True),    # very wide: 512 block columns, 32 strips per row
    (16384, 34, 10, 16, False),
    (34, 4096, 8, 32, False),    # very tall: 128 block rows of 2 columns
    (34, 4096, 8, 8, False),
])
def test_parity_extreme_shapes(W, H, bd, w, lp):
    """Degenerate and extreme aspect ratios: records against the oracle."""
    Y, U, V = synth.g_frames(29, W, H, 3, bd)
    g, r, _ = run_both(Y, U, V, bd, w, lp)
    assert_records(g, r)


def test_empty_and_single_frame():
    """n_frames = 0 is an argument error (EmptyStream); one frame gives one record with
    h = 0."""
    from paper_2304_12384_b200 import VcaError

    a = Analyzer(64, 32, 8, 16, False)
    Y, U, V = synth.g_frames(3, 64, 32, 1, 8)
    with pytest.raises(VcaError) as e:
        a.analyze(*(p[:0].cuda() for p in (Y, U, V)))
    assert e.value.code == -1
    rec = records_to_numpy(a.analyze(*planes_cuda(Y, U, V)))
    assert len(rec) == 1 and rec["poc"][0] == 0 and rec["h"][0] == 0.0


def test_concurrent_contexts_on_streams():
    """Two contexts analysing on two CUDA streams at the same time give the same records as
    one after the other (contexts share no mutable state; S:362 determinism)."""
    Y, U, V = synth.g_frames(41, 264, 176, 6, 8)
    Y2, U2, V2 = synth.g_frames(42, 264, 176, 6, 8)
    d1 = planes_cuda(Y, U, V)
    d2 = planes_cuda(Y2, U2, V2)
    seq = []
    for d in (d1, d2):
        a = Analyzer(264, 176, 8, 32, True)
        seq.append(records_to_numpy(a.analyze(*d)))
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a1, a2 = Analyzer(264, 176, 8, 32, True), Analyzer(264, 176, 8, 32, True)
    outs = []
    for _ in range(3):  # several overlapping rounds
        a1.reset(0)
        a2.reset(0)
        with torch.cuda.stream(s1):
            r1 = a1.analyze(*d1, stream=s1)
        with torch.cuda.stream(s2):
            r2 = a2.analyze(*d2, stream=s2)
        torch.cuda.synchronize()
        outs.append((records_to_numpy(r1), records_to_numpy(r2)))
    for r1, r2 in outs:
        assert r1.tobytes() == seq[0].tobytes() and r2.tobytes() == seq[1].tobytes()


@pytest.mark.parametrize("W,H,bd,w,lp", [(1024, 72, 8, 32, True), (640, 40, 10, 16, False), (1152, 70, 8, 16, True)])
def test_parity_padded_pitch_tma4(W, H, bd, w, lp):
    """4-D tensor-map geometry (row bytes a multiple of the box width) with a row pitch well above
    the row bytes and a frame stride above H x pitch: records against the oracle, production vs
    DUMP bit for bit, every block's integer checks."""
    F = 3
    Y, U, V = synth.g_frames(37, W, H, F, bd)
    padded = []
    for p in (Y, U, V):
        f, h, wd = p.shape
        buf = torch.zeros((f, h + 3, wd + 256 // p.element_size()), dtype=p.dtype, device="cuda")
        buf[:, :h, :wd] = p.cuda()
        padded.append(buf[:, :h, :wd])
    pair = Pair(W, H, bd, w, lp)
    rec, hy, ch = pair.analyze(*padded)
    ro, rhy, rch = oracle_checks(Y, U, V, bd, w, lp)
    assert_records(rec, ro)
    assert_records(rec, ro, rtol=1e-12)
    assert_checks(ch, rch)
