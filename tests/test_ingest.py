"""Host-side ingest, CSV and CLI checks (no GPU): the native Y4M / raw-YUV readers,
the features CSV writer and the summary of include/vca_io.h against SPEC.md's
ingest / stats / cli examples and against numpy
on the same bytes.  Readings R-13..R-16 where SPEC is inconsistent."""
import io
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2304_12384_b200 import vcaio
from paper_2304_12384_b200.vca import RECORD_DTYPE, VcaError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EOF = vcaio.VCA_IO_EOF


# ---------------------------------------------------------------- Y4M header
def test_header_examples():
    info, hl, w = vcaio.parse_y4m_header(b"YUV4MPEG2 W8 H8 F25:1 Ip A1:1 C420jpeg\n")
    assert (info["width"], info["height"], info["bit_depth"], info["chroma"]) == (8, 8, 8, 420)
    assert (info["fps_num"], info["fps_den"]) == (25, 1)
    assert hl == len(b"YUV4MPEG2 W8 H8 F25:1 Ip A1:1 C420jpeg\n") and w == 0
    info, _, _ = vcaio.parse_y4m_header(b"YUV4MPEG2 W16 H16 F30000:1001 C444\n")
    assert (info["width"], info["height"], info["bit_depth"], info["chroma"]) == (16, 16, 8, 444)
    assert (info["fps_num"], info["fps_den"]) == (30000, 1001)


@pytest.mark.parametrize("tag,chroma,bd", [("420jpeg", 420, 8), ("420mpeg2", 420, 8), ("420paldv", 420, 8),
                                           ("420", 420, 8), ("422", 422, 8), ("444", 444, 8),
                                           ("420p10", 420, 10), ("422p10", 422, 10), ("444p10", 444, 10)])
def test_header_chroma_tags(tag, chroma, bd):
    info, _, _ = vcaio.parse_y4m_header(b"YUV4MPEG2 W64 H32 F24:1 C" + tag.encode() + b"\n")
    assert (info["chroma"], info["bit_depth"]) == (chroma, bd)
    cw = 32 if chroma in (420, 422) else 64
    ch = 16 if chroma == 420 else 32
    es = 1 if bd == 8 else 2
    assert info["frame_bytes"] == (64 * 32 + 2 * cw * ch) * es


def test_header_default_chroma_and_x_tokens():
    info, _, w = vcaio.parse_y4m_header(b"YUV4MPEG2 W8 H8 F25:1 XYSCSS=420JPEG XCOLORRANGE=LIMITED\n")
    assert info["chroma"] == 420 and info["bit_depth"] == 8
    assert w == vcaio.WARN_X_TOKENS  # tolerated with a warning


@pytest.mark.parametrize("hdr,code", [
    (b"JUNK W8 H8\n", -11),                            # MalformedMagic
    (b"YUV4MPEG2X W8 H8 F25:1\n", -11),
    (b"YUV4MPEG2 W8 H8 F25:1 Cmono\n", -4),            # UnsupportedChroma
    (b"YUV4MPEG2 W8 H8 F25:1 C411\n", -4),
    (b"YUV4MPEG2 W8 H8 F25:1 C420p12\n", -3),          # UnsupportedBitDepth
    (b"YUV4MPEG2 W8 H8 F25:1 C420p9\n", -3),
    (b"YUV4MPEG2 W8 H8 F25:1 It\n", -15),              # interlaced rejected
    (b"YUV4MPEG2 W8 H8 F25:1 Ib\n", -15),
    (b"YUV4MPEG2 W8 F25:1\n", -12),                    # missing H
    (b"YUV4MPEG2 W8 H8\n", -12),                       # missing F
    (b"YUV4MPEG2 W8 H8 F0:1\n", -12),                  # F num > 0
    (b"YUV4MPEG2 Wx8 H8 F25:1\n", -12),                # unparsable token
    (b"YUV4MPEG2 W7 H8 F25:1\n", -12),                 # odd width, 4:2:0
    (b"YUV4MPEG2 W8 H8 F25:1 Q1\n", -12),              # unknown token
    (b"YUV4MPEG2 W8 H8 F25:1", -12),                   # no newline
])
def test_header_errors(hdr, code):
    with pytest.raises(VcaError) as e:
        vcaio.parse_y4m_header(hdr)
    assert e.value.code == code


# ---------------------------------------------------------------- readers
def frames_420(n, w, h, bd, seed=0):
    rng = np.random.default_rng(seed)
    hi = 255 if bd == 8 else 1023
    dt = np.uint8 if bd == 8 else np.uint16
    return [rng.integers(0, hi + 1, size=(n, hh, ww)).astype(dt) for (ww, hh) in ((w, h), (w // 2, h // 2),
                                                                                     (w // 2, h // 2))]


def raw_bytes(planes):
    n = planes[0].shape[0]
    return b"".join(p[t].astype(p.dtype.newbyteorder("<")).tobytes() for t in range(n) for p in planes)


def y4m_bytes(planes, w, h, bd, frame_params=b""):
    tag = b"C420jpeg" if bd == 8 else b"C420p10"
    out = [b"YUV4MPEG2 W%d H%d F25:1 Ip A1:1 " % (w, h) + tag + b"\n"]
    for t in range(planes[0].shape[0]):
        out.append(b"FRAME" + frame_params + b"\n")
        out.extend(p[t].astype(p.dtype.newbyteorder("<")).tobytes() for p in planes)
    return b"".join(out)


def test_raw_exact_one_frame(tmp_path):
    f = tmp_path / "a.yuv"
    f.write_bytes(bytes(range(96)))                     # 8x8 4:2:0 8-bit: 64 + 16 + 16 bytes
    with vcaio.Reader(str(f), "raw", 8, 8, 8) as r:
        assert r.info["frame_bytes"] == 96 and r.info["frame_count"] == 1
        rc, (Y, U, V) = r.read(4)
        assert rc == EOF and len(Y) == 1
        assert Y[0].tobytes() == bytes(range(64)) and U[0].tobytes() == bytes(range(64, 80))
        assert V[0].tobytes() == bytes(range(80, 96))
        assert r.warnings == 0


@pytest.mark.parametrize("size,frames", [(140, 1), (200, 2), (3 * 96, 3), (3 * 96 + 95, 3)])
def test_raw_trailing_partial_frame(tmp_path, size, frames):
    """R-14: a trailing partial raw frame is discarded and flagged, never half-read."""
    f = tmp_path / "a.yuv"
    f.write_bytes(bytes(i & 255 for i in range(size)))
    with vcaio.Reader(str(f), "raw", 8, 8, 8) as r:
        rc, (Y, U, V) = r.read(10)
        assert rc == EOF and len(Y) == frames == r.frames
        assert bool(r.warnings & vcaio.WARN_TRAILING_BYTES) == (size % 96 != 0)


def test_raw_10bit_little_endian(tmp_path):
    f = tmp_path / "a.yuv"
    b = bytearray(192)
    b[0:2] = bytes([0xBC, 0x02])                        # 700
    f.write_bytes(bytes(b))
    with vcaio.Reader(str(f), "raw", 8, 8, 10) as r:
        rc, (Y, U, V) = r.read(1)
        assert rc == vcaio.VCA_OK and Y.dtype == np.uint16 and Y[0, 0, 0] == 700


def test_raw_missing_file(tmp_path):
    with pytest.raises(VcaError) as e:
        vcaio.Reader(str(tmp_path / "nope.yuv"), "raw", 8, 8, 8)
    assert e.value.code == -10


@pytest.mark.parametrize("bd", [8, 10])
def test_raw_round_trip(tmp_path, bd):
    planes = frames_420(5, 40, 24, bd, seed=bd)
    f = tmp_path / "a.yuv"
    f.write_bytes(raw_bytes(planes))
    with vcaio.Reader(str(f), "raw", 40, 24, bd) as r:
        got = []
        while True:
            rc, fr = r.read(2)                            # batches straddle the end
            got.append(fr)
            if rc != vcaio.VCA_OK:
                break
        assert rc == EOF
    for p in range(3):
        assert np.array_equal(np.concatenate([g[p] for g in got]), planes[p])


@pytest.mark.parametrize("bd,params", [(8, b""), (10, b""), (8, b" Ixyz XFOO=1")])
def test_y4m_round_trip(tmp_path, bd, params):
    planes = frames_420(3, 24, 16, bd, seed=7)
    f = tmp_path / "a.y4m"
    f.write_bytes(y4m_bytes(planes, 24, 16, bd, params))
    with vcaio.Reader(str(f), "y4m") as r:
        assert r.info["bit_depth"] == bd
        assert r.info["frame_count"] == (3 if not params else -1)   # derivable only with bare markers
        rc, fr = r.read(8)
        assert rc == EOF and r.frames == 3
    for p in range(3):
        assert np.array_equal(fr[p], planes[p])


def test_y4m_two_frames_then_eof(tmp_path):
    planes = frames_420(2, 8, 8, 8)
    f = tmp_path / "a.y4m"
    f.write_bytes(y4m_bytes(planes, 8, 8, 8))
    with vcaio.Reader(str(f), "y4m") as r:
        rc, fr = r.read(1)
        assert rc == vcaio.VCA_OK and len(fr[0]) == 1
        rc, fr = r.read(1)
        assert rc == vcaio.VCA_OK and np.array_equal(fr[0][0], planes[0][1])
        rc, fr = r.read(1)
        assert rc == EOF and len(fr[0]) == 0


def test_y4m_truncated_and_bad_marker(tmp_path):
    planes = frames_420(2, 8, 8, 8)
    good = y4m_bytes(planes, 8, 8, 8)
    f = tmp_path / "t.y4m"
    f.write_bytes(good[:-10])
    with vcaio.Reader(str(f), "y4m") as r:
        rc, fr = r.read(4)
        assert rc == -13 and len(fr[0]) == 1            # frame 0 delivered, then TruncatedFrame
    f.write_bytes(good.replace(b"FRAME", b"FRAMX", 2))
    with vcaio.Reader(str(f), "y4m") as r:
        rc, fr = r.read(4)
        assert rc == -14 and len(fr[0]) == 0


def test_y4m_reader_stops_at_payload(tmp_path):
    """The reader never consumes bytes past the frames it delivered: after one
    frame, the next read sees exactly the trailing junk and reports a bad marker."""
    planes = frames_420(1, 8, 8, 8)
    f = tmp_path / "j.y4m"
    f.write_bytes(y4m_bytes(planes, 8, 8, 8) + b"JUNKJUNK")
    with vcaio.Reader(str(f), "y4m") as r:
        rc, fr = r.read(1)
        assert rc == vcaio.VCA_OK and np.array_equal(fr[0][0], planes[0][0])
        rc, fr = r.read(1)
        assert rc == -14


def test_y4m_from_pipe():
    planes = frames_420(2, 16, 8, 8, seed=3)
    data = y4m_bytes(planes, 16, 8, 8)
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2304_12384_b200 import vcaio\n"
            "r = vcaio.Reader('-', 'y4m')\n"
            "rc, fr = r.read(5)\n"
            "print(rc, r.info['frame_count'], len(fr[0]), int(fr[0].sum()))\n") % ROOT
    out = subprocess.run([sys.executable, "-c", code], input=data, capture_output=True, timeout=120)
    assert out.returncode == 0, out.stderr
    rc, count, n, s = out.stdout.split()
    assert (int(rc), int(count), int(n), int(s)) == (EOF, -1, 2, int(planes[0].astype(np.int64).sum()))


# ---------------------------------------------------------------- CSV and summary
def records(n, seed=0):
    rng = np.random.default_rng(seed)
    r = np.zeros(n, RECORD_DTYPE)
    r["poc"] = np.arange(n)
    for f in ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V"):
        r[f] = rng.uniform(0, 100, n)
    return r


def test_csv_header_only(tmp_path):
    p = tmp_path / "o.csv"
    n = vcaio.write_csv(str(p), records(0))
    assert p.read_bytes() == b"POC,E_Y,h,L_Y,E_U,L_U,E_V,L_V\n" and n == len(p.read_bytes())


def test_csv_zero_record(tmp_path):
    p = tmp_path / "o.csv"
    vcaio.write_csv(str(p), np.zeros(1, RECORD_DTYPE))
    assert p.read_bytes().split(b"\n")[1] == b"0,0.000000,0.000000,0.000000,0.000000,0.000000,0.000000,0.000000"


def test_csv_round_trip(tmp_path):
    r = records(100, seed=5)
    p = tmp_path / "o.csv"
    vcaio.write_csv(str(p), r)
    data = p.read_bytes()
    assert b"\r" not in data and data.endswith(b"\n")
    back = np.genfromtxt(io.BytesIO(data), delimiter=",", names=True)
    assert np.array_equal(back["POC"].astype(np.int64), r["poc"])
    for f in ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V"):
        assert np.max(np.abs(back[f] - r[f])) <= 5e-7 + 1e-15


def test_csv_unwritable(tmp_path):
    with pytest.raises(VcaError) as e:
        vcaio.write_csv(str(tmp_path / "no" / "such" / "dir.csv"), records(1))
    assert e.value.code == -10


def test_summary():
    r = records(1)
    mean, mx = vcaio.summarize(r)
    assert mean == mx == {f: float(r[f][0]) for f in mean}
    r = np.zeros(2, RECORD_DTYPE)
    r["E_Y"] = (1.0, 3.0)
    mean, mx = vcaio.summarize(r)
    assert mean["E_Y"] == 2.0 and mx["E_Y"] == 3.0
    r = records(100, seed=9)
    mean, mx = vcaio.summarize(r)
    for f in mean:
        s = 0.0
        for v in r[f]:                                   # POC-order re-summation
            s += float(v)
        assert mean[f] == s / 100 and mx[f] == float(r[f].max())
    with pytest.raises(VcaError):
        vcaio.summarize(np.zeros(0, RECORD_DTYPE))


# ---------------------------------------------------------------- CLI usage / input errors
def cli(*args, **kw):
    return subprocess.run([sys.executable, "-m", "paper_2304_12384_b200.cli", *args], capture_output=True, text=True,
                          cwd=ROOT, timeout=300, **kw)


def test_cli_usage_errors(tmp_path):
    f = tmp_path / "clip.yuv"
    f.write_bytes(bytes(96))
    assert cli("analyze", str(f)).returncode == 1                 # raw without --width
    assert cli().returncode == 1                                  # no subcommand
    assert cli("analyze", str(f), "--bogus").returncode == 1      # unknown flag
    assert cli("analyze", str(tmp_path / "clip.mp4")).returncode == 1  # format not inferable


def test_cli_input_errors(tmp_path):
    assert cli("analyze", str(tmp_path / "missing.y4m")).returncode == 2
    bad = tmp_path / "bad.y4m"
    bad.write_bytes(b"JUNK W8 H8\n")
    r = cli("analyze", str(bad))
    assert r.returncode == 2 and "MALFORMED_MAGIC" in r.stderr


# ---------------------------------------------------------------- native C client of the ABI
def native_cli(*args):
    from paper_2304_12384_b200 import build

    if not os.path.exists(build.CLI):
        build.build_cli()
    return subprocess.run([build.CLI, *args], capture_output=True, text=True, timeout=300)


def test_native_cli_usage_and_input_errors(tmp_path):
    assert native_cli().returncode == 1
    assert native_cli("a.yuv").returncode == 1                     # raw without geometry
    assert native_cli("a.y4m", "--bogus").returncode == 1
    assert native_cli(str(tmp_path / "missing.y4m")).returncode == 2
    bad = tmp_path / "bad.y4m"
    bad.write_bytes(b"JUNK W8 H8\n")
    r = native_cli(str(bad))
    assert r.returncode == 2 and "Y4M" in r.stderr


def test_y4m_parameterised_markers_with_fixed_size(tmp_path):
    """A Y4M whose later FRAME markers carry parameters but whose size happens to divide into
    bare-marker records: the positional reader delivers the verified prefix and continues
    sequentially (R-15)."""
    planes = frames_420(4, 16, 8, 8, seed=5)
    fb = 16 * 8 * 3 // 2
    head = b"YUV4MPEG2 W16 H8 F25:1 C420jpeg\n"
    recs = []
    for t in range(4):
        marker = b"FRAME\n" if t < 2 else b"FRAME Ip\n"
        recs.append(marker + b"".join(p[t].tobytes() for p in planes))
    data = head + b"".join(recs)
    # append a short junk record so the payload size is a multiple of a bare record (6 + fb):
    # the reader then starts in positional mode and must fall back at frame 2
    pad = (6 + fb) - (len(data) - len(head)) % (6 + fb)
    assert 6 <= pad < 6 + fb
    data += b"FRAME\n" + bytes(pad - 6)
    f = tmp_path / "p.y4m"
    f.write_bytes(data)
    with vcaio.Reader(str(f), "y4m") as r:
        got = []
        while True:
            rc, fr = r.read(8)
            got.append(fr)
            if rc != vcaio.VCA_OK or r.frames >= 4:
                break
        Y = np.concatenate([g[0] for g in got])
    assert np.array_equal(Y[:4], planes[0])


def test_y4m_first_failure_is_deterministic(tmp_path):
    """A valid Y4M whose frame 20 carries a parameterised marker, in a file whose size divides
    into bare-marker records: the positional readers (16 threads) see frame 20 as the end of the
    fixed-size run and every later record as misaligned; the first failing frame and its own
    status must win together (one packed atomic), so every read falls back to the sequential
    reader at frame 20 and delivers all 64 frames -- never the misaligned records' status."""
    F = 64
    planes = frames_420(F, 16, 8, 8, seed=9)
    fb = 16 * 8 * 3 // 2
    head = b"YUV4MPEG2 W16 H8 F25:1 C420jpeg\n"
    recs = [(b"FRAME Ip\n" if t == 20 else b"FRAME\n") + b"".join(p[t].tobytes() for p in planes) for t in range(F)]
    data = head + b"".join(recs)
    pad = (6 + fb) - (len(data) - len(head)) % (6 + fb)
    data += b"FRAME\n" + bytes(pad - 6)
    f = tmp_path / "race.y4m"
    f.write_bytes(data)
    for _ in range(20):
        with vcaio.Reader(str(f), "y4m") as r:
            got = []
            while r.frames < F:
                rc, fr = r.read(F - r.frames)
                assert rc == vcaio.VCA_OK, (rc, r.frames)
                got.append(fr[0])
            Y = np.concatenate(got)
        assert np.array_equal(Y[:F], planes[0])
