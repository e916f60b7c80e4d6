"""GPU checks of the streaming path (include/vca_io.h, NEXT-3): a Y4M / raw file read
by the native reader thread into pinned batches and analysed with overlapped H2D
(vca_analyze_stream) gives records bit-identical to the device-resident path on
the same bytes and within the parity bar of the CPU oracle; the CLI writes the
same CSV."""
import re

import numpy as np
import pytest
import torch

import oracle
from paper_2304_12384_b200 import Analyzer, records_to_numpy, synth, vcaio
from paper_2304_12384_b200.vca import RECORD_DTYPE

from test_ingest import cli, raw_bytes, y4m_bytes
from test_parity_gpu import assert_records

pytestmark = pytest.mark.gpu


def device_records(planes_np, bd, w, lp):
    t = [torch.from_numpy(p.view(np.int16) if p.dtype == np.uint16 else p) for p in planes_np]
    a = Analyzer(planes_np[0].shape[2], planes_np[0].shape[1], bd, w, lp)
    rec = a.analyze(*synth.with_pitch(tuple(x.cuda() for x in t)))
    torch.cuda.synchronize()
    return records_to_numpy(rec)


def gen(n, W, H, bd, seed):
    Y, U, V = synth.g_frames(seed, W, H, n, bd)
    return list(synth.as_numpy_planes(Y, U, V))


@pytest.mark.parametrize("W,H,bd,w,lp,batch", [(200, 136, 8, 32, True, 5), (200, 136, 8, 32, False, 32),
                                               (136, 100, 10, 16, False, 4), (264, 176, 8, 16, False, 7)])
def test_stream_y4m_equals_device_path_and_oracle(tmp_path, W, H, bd, w, lp, batch):
    planes = gen(17, W, H, bd, seed=W + bd)
    f = tmp_path / "clip.y4m"
    f.write_bytes(y4m_bytes(planes, W, H, bd))
    with vcaio.Reader(str(f), "y4m") as r:
        a = Analyzer(W, H, bd, w, lp)
        rec, secs = vcaio.analyze_stream(a, r, batch_frames=batch)
    assert len(rec) == 17 and secs > 0
    dev = device_records(planes, bd, w, lp)
    assert rec.tobytes() == dev.tobytes()                 # bit-identical to the device-resident path
    ref = oracle.analyze(*planes, bd, w, lp)
    assert_records(rec, ref)


def test_stream_capacity_chunks_and_raw(tmp_path):
    """Several vca_analyze_stream calls (capacity < frames) continue the sequence (carried
    H_Y, POC) exactly like one call; the raw reader gives the same records."""
    W, H = 200, 136
    planes = gen(13, W, H, 8, seed=3)
    f = tmp_path / "clip.yuv"
    f.write_bytes(raw_bytes(planes) + b"\x01\x02")    # trailing partial frame: discarded
    with vcaio.Reader(str(f), "raw", W, H, 8) as r:
        assert r.warnings & vcaio.WARN_TRAILING_BYTES
        a = Analyzer(W, H, 8, 32, True)
        rec, _ = vcaio.analyze_stream(a, r, batch_frames=3, capacity=4)
    dev = device_records(planes, 8, 32, True)
    assert rec.tobytes() == dev.tobytes()


def test_stream_geometry_mismatch(tmp_path):
    planes = gen(2, 64, 32, 8, seed=1)
    f = tmp_path / "clip.y4m"
    f.write_bytes(y4m_bytes(planes, 64, 32, 8))
    with vcaio.Reader(str(f), "y4m") as r:
        a = Analyzer(128, 32, 8, 16, False)
        with pytest.raises(Exception) as e:
            vcaio.analyze_stream(a, r)
        assert getattr(e.value, "code", None) == -5


def test_cli_analyze_and_bench(tmp_path):
    W, H = 200, 136
    planes = gen(9, W, H, 8, seed=11)
    f = tmp_path / "clip.y4m"
    f.write_bytes(y4m_bytes(planes, W, H, 8))
    out = tmp_path / "out.csv"
    r = cli("analyze", str(f), "-o", str(out), "--block-size", "32", "--low-pass", "--batch-frames", "4")
    assert r.returncode == 0, r.stderr
    assert "# mean" in r.stderr
    dev = device_records(planes, 8, 32, True)
    want = tmp_path / "want.csv"
    vcaio.write_csv(str(want), dev)
    assert out.read_bytes() == want.read_bytes()          # identical CSV bytes
    back = np.genfromtxt(str(out), delimiter=",", names=True)
    ref = oracle.analyze(*planes, 8, 32, True)
    for k in ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V"):
        assert np.max(np.abs(back[k] - ref[k])) <= 5e-7 + 1e-6 * np.max(np.abs(ref[k]))
    # repeat: byte-identical output
    out2 = tmp_path / "out2.csv"
    assert cli("analyze", str(f), "-o", str(out2), "--block-size", "32", "--low-pass").returncode == 0
    assert out2.read_bytes() == out.read_bytes()
    # bench: the fps line and no CSV
    b = cli("bench", str(f), "--block-size", "32", "--low-pass")
    assert b.returncode == 0, b.stderr
    assert re.fullmatch(r"frames=9 seconds=[0-9.]+ fps=[0-9]+\.[0-9]{2}\n", b.stdout)


def test_cli_constant_clip(tmp_path):
    """a 3-frame constant clip -> 3 rows, all E and h zero."""
    W, H = 64, 64
    planes = [np.full((3, H, W), 128, np.uint8), np.full((3, H // 2, W // 2), 100, np.uint8),
              np.full((3, H // 2, W // 2), 200, np.uint8)]
    f = tmp_path / "const.y4m"
    f.write_bytes(y4m_bytes(planes, W, H, 8))
    out = tmp_path / "c.csv"
    r = cli("analyze", str(f), "-o", str(out))
    assert r.returncode == 0, r.stderr
    back = np.genfromtxt(str(out), delimiter=",", names=True)
    assert len(back) == 3
    for k in ("E_Y", "h", "E_U", "E_V"):
        assert np.all(back[k] == 0.0)


def test_native_cli_matches_python_cli(tmp_path):
    """The plain-C client (csrc/vca_cli.c, no Python/PyTorch) writes the same CSV bytes."""
    from test_ingest import native_cli

    W, H = 264, 176
    planes = gen(7, W, H, 8, seed=23)
    f = tmp_path / "clip.y4m"
    f.write_bytes(y4m_bytes(planes, W, H, 8))
    a, b = tmp_path / "py.csv", tmp_path / "c.csv"
    assert cli("analyze", str(f), "-o", str(a), "--block-size", "32", "--low-pass").returncode == 0
    r = native_cli(str(f), "-o", str(b), "--block", "32", "--low-pass", "--batch", "3")
    assert r.returncode == 0, r.stderr
    assert a.read_bytes() == b.read_bytes()


def test_native_cli_raw_10bit(tmp_path):
    """Raw 10-bit little-endian input through the plain-C client vs the device-resident path."""
    from test_ingest import native_cli

    W, H = 136, 100
    planes = gen(5, W, H, 10, seed=31)
    f = tmp_path / "clip.yuv"
    f.write_bytes(raw_bytes(planes))
    out = tmp_path / "c.csv"
    r = native_cli(str(f), "--width", str(W), "--height", str(H), "--bit-depth", "10", "--block", "16", "-o", str(out))
    assert r.returncode == 0, r.stderr
    want = tmp_path / "want.csv"
    vcaio.write_csv(str(want), device_records(planes, 10, 16, False))
    assert out.read_bytes() == want.read_bytes()
