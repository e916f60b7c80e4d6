"""ctypes binding of libvca's ingest / streaming / CSV calls (include/vca_io.h) --
argument marshalling only; the readers, the streaming driver and the CSV writer
are native (csrc/vca_io.cpp).  SURVEY.md §8(f) NEXT-3; SPEC.md ingest S:24-93,
stats S:402-469."""
from __future__ import annotations

import ctypes

import numpy as np

from .vca import CHROMA, RECORD_DTYPE, VCA_OK, Analyzer, VcaError, lib

VCA_IO_EOF = 1
WARN_TRAILING_BYTES = 1
WARN_X_TOKENS = 2
CHROMA_NAME = {0: 420, 1: 422, 2: 444}


class StreamInfo(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("bit_depth", ctypes.c_int),
                ("chroma_format", ctypes.c_int), ("fps_num", ctypes.c_int), ("fps_den", ctypes.c_int),
                ("bytes_per_sample", ctypes.c_int), ("chroma_width", ctypes.c_int),
                ("chroma_height", ctypes.c_int), ("frame_bytes", ctypes.c_int64), ("frame_count", ctypes.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["chroma"] = CHROMA_NAME.get(self.chroma_format, self.chroma_format)
        return d


def parse_y4m_header(data: bytes):
    """Y4M header bytes -> (info dict, header length, warning bits); raises VcaError."""
    info = StreamInfo()
    hl = ctypes.c_size_t()
    w = ctypes.c_int()
    rc = lib().vca_y4m_parse_header(data, len(data), ctypes.byref(info), ctypes.byref(hl), ctypes.byref(w))
    if rc != VCA_OK:
        raise VcaError(rc, "vca_y4m_parse_header")
    return info.as_dict(), hl.value, w.value


class Reader:
    """A Y4M or raw-YUV frame source (vca_y4m_open / vca_raw_open ... vca_reader_close)."""

    def __init__(self, path: str, fmt: str = "y4m", width: int = 0, height: int = 0, bit_depth: int = 8,
                 chroma: int = 420):
        self._L = lib()
        h = ctypes.c_void_p()
        info = StreamInfo()
        if fmt == "y4m":
            rc = self._L.vca_y4m_open(path.encode(), ctypes.byref(h), ctypes.byref(info))
        elif fmt == "raw":
            rc = self._L.vca_raw_open(path.encode(), width, height, bit_depth, CHROMA.get(chroma, 99),
                                      ctypes.byref(h), ctypes.byref(info))
        else:
            raise ValueError("format must be 'y4m' or 'raw'")
        if rc != VCA_OK:
            raise VcaError(rc, "vca_%s_open" % ("y4m" if fmt == "y4m" else "raw"))
        self._h = h
        self.info = info.as_dict()

    def close(self):
        if getattr(self, "_h", None):
            self._L.vca_reader_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def frames(self) -> int:
        return int(self._L.vca_reader_frames(self._h))

    @property
    def warnings(self) -> int:
        return int(self._L.vca_reader_warnings(self._h))

    def read(self, max_frames: int):
        """-> (status, [Y, U, V] numpy arrays [n][h][w] (uint8 / uint16)); status VCA_OK,
        VCA_IO_EOF or a negative code (frames before it are returned)."""
        i = self.info
        dt = np.uint8 if i["bytes_per_sample"] == 1 else np.uint16
        dims = ((i["height"], i["width"]), (i["chroma_height"], i["chroma_width"]),
                (i["chroma_height"], i["chroma_width"]))
        bufs = [np.zeros((max_frames,) + d, dt) for d in dims]
        es = np.dtype(dt).itemsize
        P3 = ctypes.c_void_p * 3
        I3 = ctypes.c_int64 * 3
        n = ctypes.c_int()
        rc = self._L.vca_reader_read(self._h, max_frames, P3(*[b.ctypes.data for b in bufs]),
                                     I3(*[d[1] * es for d in dims]), I3(*[d[0] * d[1] * es for d in dims]),
                                     ctypes.byref(n))
        return rc, [b[:n.value] for b in bufs]


def analyze_stream(analyzer: Analyzer, reader: Reader, batch_frames: int = 32, capacity: int | None = None):
    """Stream a whole source through a context (vca_analyze_stream, called until
    the source is exhausted) -> (structured records, seconds); raises VcaError."""
    L = lib()
    chunks = []
    total_s = 0.0
    cap = capacity or (reader.info["frame_count"] if reader.info["frame_count"] > 0 else 1024)
    while True:
        out = np.zeros(cap, dtype=RECORD_DTYPE)
        n = ctypes.c_int64()
        sec = ctypes.c_double()
        rc = L.vca_analyze_stream(analyzer._h, reader._h, batch_frames, out.ctypes.data, cap, ctypes.byref(n),
                                  ctypes.byref(sec))
        total_s += sec.value
        chunks.append(out[:n.value])
        if rc == VCA_IO_EOF:
            break
        if rc != VCA_OK:
            raise VcaError(rc, "vca_analyze_stream")
    return np.concatenate(chunks), total_s


def write_csv(path: str, records: np.ndarray) -> int:
    """Features CSV (S:456 format) -> bytes written; raises VcaError."""
    rec = np.ascontiguousarray(records, dtype=RECORD_DTYPE)
    n = lib().vca_write_csv(path.encode(), rec.ctypes.data if len(rec) else None, len(rec))
    if n < 0:
        raise VcaError(int(n), "vca_write_csv")
    return int(n)


def summarize(records: np.ndarray):
    """-> (mean, max) dicts per feature (vca_summarize, POC-order sums)."""
    rec = np.ascontiguousarray(records, dtype=RECORD_DTYPE)
    mean = np.zeros(7)
    mx = np.zeros(7)
    rc = lib().vca_summarize(rec.ctypes.data if len(rec) else None, len(rec), mean.ctypes.data, mx.ctypes.data)
    if rc != VCA_OK:
        raise VcaError(rc, "vca_summarize")
    names = ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V")
    return dict(zip(names, mean.tolist())), dict(zip(names, mx.tolist()))
