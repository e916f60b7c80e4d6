"""CPU oracle for the VCA v2.0 hot path (arxiv 2304.12384) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product path
(``paper_2304_12384_b200``) never imports it and shares no code with it.

The arithmetic lives in ``vca_oracle.c`` (plain C, int64 / double, sequential
raster-order sums, OpenMP over frames only); this module is argument
marshalling plus the gcc build.  Every function is pinned by
``tests/test_oracle_*.py``; see DESIGN.md "Oracle and pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vca_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

RECORD_DTYPE = np.dtype(
    [("poc", "<i8"), ("E_Y", "<f8"), ("h", "<f8"), ("L_Y", "<f8"), ("E_U", "<f8"),
     ("L_U", "<f8"), ("E_V", "<f8"), ("L_V", "<f8")]
)
FEATURES = ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V")


def build(force: bool = False) -> str:
    """Compile vca_oracle.c with gcc (-O2, OpenMP, no -march) into liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-Wextra", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.vo_basis.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int32)]
        L.vo_weight.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.vo_weight.restype = ctypes.c_double
        L.vo_block.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p, i64p,
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.vo_resolve_block.argtypes = [ctypes.c_int, ctypes.c_int]
        L.vo_chroma_block.argtypes = [ctypes.c_int]
        L.vo_block_count.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.vo_block_count.restype = ctypes.c_int64
        L.vo_analyze.argtypes = [ctypes.POINTER(ctypes.c_void_p), i64p, i64p, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_int]
        P3 = ctypes.c_void_p * 3
        L.vo_analyze_checks.argtypes = L.vo_analyze.argtypes + [P3, P3, P3]
        _lib = L
    return _lib


def basis(n: int) -> np.ndarray:
    T = np.zeros((n, n), dtype=np.int32)
    rc = lib().vo_basis(n, T.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    if rc:
        raise ValueError("vo_basis(%d) -> %d" % (n, rc))
    return T


def weight(n: int, i: int, j: int) -> float:
    return lib().vo_weight(n, i, j)


def resolve_block(height: int, block_size: int) -> int:
    return lib().vo_resolve_block(height, block_size)


def chroma_block(w: int) -> int:
    return lib().vo_chroma_block(w)


def block_count(pw: int, ph: int, w: int) -> int:
    return lib().vo_block_count(pw, ph, w)


def _plane_u8(plane: np.ndarray):
    """A 2-D uint8 or uint16 plane -> (byte pointer holder, pitch, width in samples)."""
    plane = np.ascontiguousarray(plane)
    if plane.dtype not in (np.uint8, np.uint16):
        raise TypeError("planes are uint8 (8-bit) or little-endian uint16 (10-bit)")
    return plane, plane.strides[0], plane.shape[1]


def block(plane: np.ndarray, bd: int, w: int, lowpass: bool, r: int, c: int):
    """Steps 1-4 for one block: returns (coeffs int64 [n][n], sumx, H, L)."""
    plane, pitch, pw = _plane_u8(plane)
    ph = plane.shape[0]
    n = w // 2 if lowpass else w
    coeffs = np.zeros((n, n), dtype=np.int64)
    sumx = ctypes.c_int64()
    H = ctypes.c_double()
    L = ctypes.c_double()
    rc = lib().vo_block(plane.ctypes.data, pitch, bd, pw, ph, w, int(bool(lowpass)), r, c,
                        coeffs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ctypes.byref(sumx),
                        ctypes.byref(H), ctypes.byref(L))
    if rc:
        raise ValueError("vo_block -> %d" % rc)
    return coeffs, sumx.value, H.value, L.value


def analyze(Y: np.ndarray, U: np.ndarray, V: np.ndarray, bit_depth: int, block_size: int, lowpass: bool,
            n_halo: int = 0, prev_HY: np.ndarray | None = None, first_poc: int = 0,
            want_HY: bool = False, n_threads: int = 0, want_checks: bool = False):
    """Analyse frames [F][H][W] (Y) and [F][H/2][W/2] (U, V).

    Returns the structured record array (RECORD_DTYPE) for frames n_halo..F-1,
    with ``want_HY`` also the per-block luma energies [F][C_Y], and with
    ``want_checks`` also, per plane, {"chk", "sumx", "H"} arrays [F][C_p] of every
    block's AC checksum sum_{(i,j)!=(0,0)} C_ij (i n + j + 1), sample sum and H.
    """
    planes = [np.ascontiguousarray(p) for p in (Y, U, V)]
    for p in planes:
        if p.ndim != 3:
            raise ValueError("planes are [frames][rows][cols]")
    F, height, width = planes[0].shape
    if planes[0].dtype == np.uint16:
        assert bit_depth == 10
    ptrs = (ctypes.c_void_p * 3)(*[p.ctypes.data for p in planes])
    pitch = (ctypes.c_int64 * 3)(*[p.strides[1] for p in planes])
    fstride = (ctypes.c_int64 * 3)(*[p.strides[0] for p in planes])
    n_out = F - n_halo
    out = np.zeros(max(n_out, 0), dtype=RECORD_DTYPE)
    w = resolve_block(height, block_size)
    CY = block_count(width, height, w)
    HY = np.zeros((F, CY), dtype=np.float64) if want_HY else None
    prev = None
    if prev_HY is not None:
        prev = np.ascontiguousarray(prev_HY, dtype=np.float64)
        assert prev.shape == (CY,)
    checks = None
    args = [ptrs, pitch, fstride, width, height, bit_depth, block_size, int(bool(lowpass)),
            F, n_halo, None if prev is None else prev.ctypes.data, first_poc,
            out.ctypes.data, None if HY is None else HY.ctypes.data, n_threads]
    if want_checks:
        wc = chroma_block(w)
        counts = [CY, block_count(width // 2, height // 2, wc), block_count(width // 2, height // 2, wc)]
        checks = [{"chk": np.zeros((F, c), np.int64), "sumx": np.zeros((F, c), np.int64),
                   "H": np.zeros((F, c), np.float64)} for c in counts]
        P3 = ctypes.c_void_p * 3
        rc = lib().vo_analyze_checks(*args, P3(*[d["chk"].ctypes.data for d in checks]),
                                     P3(*[d["sumx"].ctypes.data for d in checks]),
                                     P3(*[d["H"].ctypes.data for d in checks]))
    else:
        rc = lib().vo_analyze(*args)
    if rc:
        raise ValueError("vo_analyze -> %d" % rc)
    res = [out]
    if want_HY:
        res.append(HY)
    if want_checks:
        res.append(checks)
    return res[0] if len(res) == 1 else tuple(res)
