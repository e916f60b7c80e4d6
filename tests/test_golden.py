"""Golden fixtures (tests/golden/): SPEC.md's printed examples (spec_examples.json, each
with its line) and values derived from the definitions alone by make_golden.py
(derived.json: basis fingerprints, the S:197-199 checkerboard constant, the frame-level
closed form).  Checked here against the CPU oracle and the host-side ingest / CSV code;
tests/test_parity_gpu.py::test_golden_closed_form_gpu checks the CUDA path."""
import json
import os

import numpy as np
import pytest

from paper_2304_12384_b200 import vcaio
from paper_2304_12384_b200.vca import RECORD_DTYPE, VcaError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
DER = json.load(open(os.path.join(GOLD, "derived.json")))


@pytest.mark.parametrize("n", (4, 8, 16, 32))
def test_basis_fingerprints(oracle_mod, n):
    T = oracle_mod.basis(n).astype(np.int64)
    f = DER["basis"][str(n)]
    assert int(np.abs(T).sum()) == f["sum_abs"] and int((T * T).sum()) == f["sum_sq"]
    assert T[1].tolist() == f["row1"]


def test_checkerboard_constant(oracle_mod):
    X = np.array([[255 * ((x + y) % 2) for x in range(8)] for y in range(8)], np.uint8)
    H = oracle_mod.block(X, 8, 8, False, 0, 0)[2]
    assert H == pytest.approx(DER["checkerboard_8x8_H"]["value"], rel=1e-13)


@pytest.mark.parametrize("mode", ("full", "lowpass"))
def test_closed_form_frames(oracle_mod, mode):
    from test_oracle_pins import _fixture_frames

    g = DER["closed_form_frames"][mode]
    Y, U, V = _fixture_frames((50, 20), mode == "lowpass")
    rec = oracle_mod.analyze(Y, U, V, 8, 32, mode == "lowpass")
    assert rec["E_Y"].tolist() == pytest.approx(g["E_Y"], rel=1e-14)
    assert rec["h"].tolist() == pytest.approx(g["h"], rel=1e-14, abs=0)
    for f in ("L_Y", "L_U", "L_V"):
        assert rec[f].tolist() == pytest.approx([g[f]] * 2, rel=1e-15)
    assert np.all(rec["E_U"] == 0.0) and np.all(rec["E_V"] == 0.0)


def block_of(desc):
    if desc.startswith("constant 8x8 v="):
        return np.full((8, 8), int(desc.split("=")[1]), np.uint8)
    if desc.startswith("constant 16x16 v="):
        return np.full((16, 16), int(desc.split("=")[1]), np.uint8)
    if desc == "all-zero 8x8":
        return np.zeros((8, 8), np.uint8)
    if desc == "impulse 8x8 at (0,0)":
        X = np.zeros((8, 8), np.uint8)
        X[0, 0] = 1
        return X
    if desc == "8x8, rows identical":
        return np.tile(np.arange(8, dtype=np.uint8) * 30, (8, 1))
    if desc.startswith("2x2 tile"):
        return np.tile(np.array([[10, 20], [30, 40]], np.uint8), (4, 4))
    if desc.startswith("checkerboard"):
        return np.array([[255 * ((x + y) % 2) for x in range(8)] for y in range(8)], np.uint8)
    raise KeyError(desc)


@pytest.mark.parametrize("ex", SPEC["dct"], ids=[e["cite"] for e in SPEC["dct"]])
def test_spec_dct(oracle_mod, ex):
    X = block_of(ex["block"])
    n = X.shape[0]
    C, _, _, _ = oracle_mod.block(X, 8, n, False, 0, 0)
    if "orthonormal_dc" in ex:                      # R-2: C / (4096 n) is the orthonormal scale
        assert C[0, 0] / (4096.0 * n) == ex["orthonormal_dc"]
    if ex.get("ac") == 0:
        assert np.all(C.ravel()[1:] == 0)
    if ex.get("vertical_ac_zero"):
        assert np.all(C[1:, :] == 0)


@pytest.mark.parametrize("ex", SPEC["downsample"], ids=[e["cite"] for e in SPEC["downsample"]])
def test_spec_downsample(oracle_mod, ex):
    C, sumx, H, _ = oracle_mod.block(block_of(ex["block"]), 8, 8, True, 0, 0)
    assert sumx == 16 * ex["out"] and H == 0.0 and np.all(C.ravel()[1:] == 0)


@pytest.mark.parametrize("ex", SPEC["luminescence"], ids=[e["cite"] for e in SPEC["luminescence"]])
def test_spec_luminescence(oracle_mod, ex):
    X = block_of(ex["block"])
    assert oracle_mod.block(X, 8, X.shape[0], False, 0, 0)[3] == ex["L"]


@pytest.mark.parametrize("ex", SPEC["y4m_header"], ids=[e["cite"] for e in SPEC["y4m_header"]])
def test_spec_y4m_header(ex):
    if "error" in ex:
        with pytest.raises(VcaError) as e:
            vcaio.parse_y4m_header(ex["header"].encode())
        assert ex["error"] in str(e.value)
        return
    info, _, _ = vcaio.parse_y4m_header(ex["header"].encode())
    assert (info["width"], info["height"], info["bit_depth"], info["chroma"]) == (
        ex["width"], ex["height"], ex["bit_depth"], ex["chroma"])
    assert [info["fps_num"], info["fps_den"]] == ex["fps"]


def test_spec_raw_10bit(tmp_path):
    ex = SPEC["raw_10bit"][0]
    f = tmp_path / "a.yuv"
    f.write_bytes(bytes.fromhex(ex["bytes_hex"]) + bytes(190))
    with vcaio.Reader(str(f), "raw", 8, 8, 10) as r:
        rc, (Y, _, _) = r.read(1)
        assert Y[0, 0, 0] == ex["sample"]


def test_spec_csv(tmp_path):
    p = tmp_path / "o.csv"
    vcaio.write_csv(str(p), np.zeros(0, RECORD_DTYPE))
    assert p.read_text() == SPEC["csv"][0]["text"]
    vcaio.write_csv(str(p), np.zeros(1, RECORD_DTYPE))
    assert p.read_text().splitlines()[1] == SPEC["csv"][1]["row"]


def test_spec_summary():
    ex = SPEC["summary"][0]
    r = np.zeros(len(ex["E_Y"]), RECORD_DTYPE)
    r["E_Y"] = ex["E_Y"]
    mean, mx = vcaio.summarize(r)
    assert mean["E_Y"] == ex["mean"] and mx["E_Y"] == ex["max"]
