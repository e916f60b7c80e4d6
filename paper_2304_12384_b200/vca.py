"""ctypes binding of libvca (include/vca.h) -- argument marshalling only.

Every step of the hot path runs in libvca's CUDA kernels; PyTorch supplies
device memory and streams.  There is no CPU fallback: if libvca.so cannot be
loaded (or built with nvcc) the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

VCA_OK = 0
STATUS = {
    0: "VCA_OK", -1: "VCA_ERR_INVALID_ARG", -2: "VCA_ERR_UNSUPPORTED_BLOCK_SIZE",
    -3: "VCA_ERR_UNSUPPORTED_BIT_DEPTH", -4: "VCA_ERR_UNSUPPORTED_CHROMA", -5: "VCA_ERR_GEOMETRY",
    -6: "VCA_ERR_ALIGNMENT", -7: "VCA_ERR_CUDA", -8: "VCA_ERR_OOM", -9: "VCA_ERR_SCRATCH",
    1: "VCA_IO_EOF", -10: "VCA_ERR_IO", -11: "VCA_ERR_MALFORMED_MAGIC", -12: "VCA_ERR_MALFORMED_HEADER",
    -13: "VCA_ERR_TRUNCATED_FRAME", -14: "VCA_ERR_MALFORMED_FRAME_MARKER", -15: "VCA_ERR_INTERLACED",
}
PATHS = {1: "fused_mma", 2: "warp_generic"}
CHROMA = {420: 0, 422: 1, 444: 2}

RECORD_DTYPE = np.dtype(
    [("poc", "<i8"), ("E_Y", "<f8"), ("h", "<f8"), ("L_Y", "<f8"), ("E_U", "<f8"),
     ("L_U", "<f8"), ("E_V", "<f8"), ("L_V", "<f8")]
)
FEATURES = ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V")

# every symbol include/vca.h and include/vca_io.h declare
EXPORTS = ("vca_create", "vca_get_info", "vca_scratch_bytes", "vca_analyze", "vca_analyze_host", "vca_reset",
           "vca_profile_enable", "vca_profile_read", "vca_debug_dump", "vca_debug_analyze", "vca_debug_mutate",
           "vca_destroy", "vca_status_string", "vca_version",
           "vca_y4m_parse_header", "vca_y4m_open", "vca_raw_open", "vca_reader_read", "vca_reader_frames",
           "vca_reader_warnings", "vca_reader_close", "vca_analyze_stream", "vca_write_csv", "vca_summarize")


class VcaError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__("%s failed: %s (%d)" % (what, STATUS.get(code, "?"), code))
        self.code = code


class _Info(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("bit_depth", ctypes.c_int),
                ("lowpass", ctypes.c_int), ("block", ctypes.c_int * 3), ("n", ctypes.c_int * 3),
                ("cols", ctypes.c_int * 3), ("rows", ctypes.c_int * 3), ("count", ctypes.c_int64 * 3),
                ("path", ctypes.c_int)]


_lib = None


def lib():
    """Load libvca.so (building it with nvcc if stale); raises if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("VCA_LIB")  # A/B experiments: an alternative build of the same sources
    if not path:
        path = _build.LIB
        if _build.stale():
            path = _build.build()
    L = ctypes.CDLL(path)
    vp, i64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    P3 = ctypes.c_void_p * 3
    I3 = ctypes.c_int64 * 3
    L.vca_create.argtypes = [c_int, c_int, c_int, c_int, c_int, c_int, ctypes.POINTER(vp)]
    L.vca_get_info.argtypes = [vp, ctypes.POINTER(_Info)]
    L.vca_scratch_bytes.argtypes = [vp, c_int]
    L.vca_scratch_bytes.restype = ctypes.c_size_t
    L.vca_analyze.argtypes = [vp, P3, I3, I3, c_int, c_int, vp, ctypes.c_size_t, vp, vp]
    L.vca_analyze_host.argtypes = [vp, P3, I3, I3, c_int, c_int, c_int, vp, vp]
    L.vca_reset.argtypes = [vp, i64]
    L.vca_profile_enable.argtypes = [vp, c_int]
    L.vca_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(i64)]
    L.vca_debug_dump.argtypes = [vp, P3, I3, P3, P3, P3, P3]
    L.vca_debug_analyze.argtypes = [vp, P3, I3, I3, c_int, c_int, vp, ctypes.c_size_t, vp, P3, P3, P3, vp]
    L.vca_debug_mutate.argtypes = [c_int, i64, c_int, c_int]
    L.vca_destroy.argtypes = [vp]
    L.vca_destroy.restype = None
    L.vca_status_string.argtypes = [c_int]
    L.vca_status_string.restype = ctypes.c_char_p
    L.vca_version.restype = ctypes.c_char_p
    # include/vca_io.h
    cp, sz = ctypes.c_char_p, ctypes.c_size_t
    L.vca_y4m_parse_header.argtypes = [cp, sz, vp, ctypes.POINTER(sz), ctypes.POINTER(c_int)]
    L.vca_y4m_open.argtypes = [cp, ctypes.POINTER(vp), vp]
    L.vca_raw_open.argtypes = [cp, c_int, c_int, c_int, c_int, ctypes.POINTER(vp), vp]
    L.vca_reader_read.argtypes = [vp, c_int, P3, I3, I3, ctypes.POINTER(c_int)]
    L.vca_reader_frames.argtypes = [vp]
    L.vca_reader_frames.restype = i64
    L.vca_reader_warnings.argtypes = [vp]
    L.vca_reader_close.argtypes = [vp]
    L.vca_reader_close.restype = None
    L.vca_analyze_stream.argtypes = [vp, vp, c_int, vp, i64, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double)]
    L.vca_write_csv.argtypes = [cp, vp, i64]
    L.vca_write_csv.restype = i64
    L.vca_summarize.argtypes = [vp, i64, vp, vp]
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc != VCA_OK:
        raise VcaError(rc, what)


def _plane_args(planes, device: bool):
    """(Y, U, V) [F][H][W] tensors -> (pointers, pitches, frame strides) in bytes."""
    import torch

    ptrs, pitch, fstride = [], [], []
    for p in planes:
        if not isinstance(p, torch.Tensor):
            raise TypeError("planes must be torch tensors")
        if device and p.device.type != "cuda":
            raise ValueError("vca_analyze takes device-resident planes (use analyze_host for host memory)")
        if not device and p.device.type != "cpu":
            raise ValueError("analyze_host takes host planes")
        if p.dim() == 2:
            p = p.unsqueeze(0)
        if p.dim() != 3 or p.stride(2) != 1:
            raise ValueError("planes are [frames][rows][cols] with unit column stride")
        es = p.element_size()
        ptrs.append(p.data_ptr())
        pitch.append(p.stride(1) * es)
        fstride.append(p.stride(0) * es)
    return ((ctypes.c_void_p * 3)(*ptrs), (ctypes.c_int64 * 3)(*pitch), (ctypes.c_int64 * 3)(*fstride))


def records_to_numpy(rec) -> np.ndarray:
    """[n, 8] float64 record tensor (device or host) -> structured numpy array."""
    a = rec.detach().cpu().contiguous().numpy() if hasattr(rec, "detach") else np.ascontiguousarray(rec)
    return a.view(np.uint8).view(RECORD_DTYPE).reshape(-1)


class Analyzer:
    """One libvca context (vca_create ... vca_destroy)."""

    def __init__(self, width: int, height: int, bit_depth: int = 8, block_size: int = 0, lowpass: bool = False,
                 chroma: int = 420):
        self._L = lib()
        h = ctypes.c_void_p()
        _check(self._L.vca_create(width, height, bit_depth, CHROMA.get(chroma, 99), block_size, int(bool(lowpass)),
                                  ctypes.byref(h)), "vca_create")
        self._h = h
        inf = _Info()
        _check(self._L.vca_get_info(self._h, ctypes.byref(inf)), "vca_get_info")
        self.info = {
            "width": inf.width, "height": inf.height, "bit_depth": inf.bit_depth, "lowpass": bool(inf.lowpass),
            "block": list(inf.block), "n": list(inf.n), "cols": list(inf.cols), "rows": list(inf.rows),
            "count": list(inf.count), "path": PATHS.get(inf.path, str(inf.path)),
        }
        self._scratch = None
        self._args_key = None        # analyze(): the plane tensors of the last call, and
        self._args = None            # their marshalled pointers / pitches / frame strides
        self._scratch_need = {}      # n_frames -> vca_scratch_bytes

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._L.vca_destroy(self._h)
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

    def _check_planes(self, planes):
        """The tensors must cover the context's planes (the library trusts the geometry it was
        created with and would read past a smaller buffer)."""
        es = 1 if self.info["bit_depth"] == 8 else 2
        W, H = self.info["width"], self.info["height"]
        for p, t in enumerate(planes):
            h, w = (H, W) if p == 0 else (H // 2, W // 2)
            if t.element_size() != es or t.shape[-2] < h or t.shape[-1] < w:
                raise ValueError("plane %d: need >= %dx%d samples of %d byte(s), got shape %s dtype %s"
                                 % (p, w, h, es, tuple(t.shape), t.dtype))
            if t.dim() == 3 and t.shape[0] != planes[0].shape[0]:
                raise ValueError("planes disagree on the number of frames")

    # -- API
    def scratch_bytes(self, max_frames: int) -> int:
        return int(self._L.vca_scratch_bytes(self._h, max_frames))

    def reset(self, next_poc: int = 0):
        _check(self._L.vca_reset(self._h, next_poc), "vca_reset")

    def analyze(self, Y, U, V, n_halo: int = 0, out=None, scratch=None, stream=None):
        """Device planes -> device records tensor [n_frames - n_halo, 8] (float64 view of vca_features)."""
        import torch

        # marshalled plane arguments are reused while the same tensor views come back (a
        # streaming caller re-analysing one buffer pays the checks and ctypes arrays once)
        key = (Y.data_ptr(), U.data_ptr(), V.data_ptr(), Y.shape, Y.stride(), U.shape, U.stride(), V.shape,
               V.stride(), Y.dtype, U.dtype, V.dtype, Y.device)
        if self._args_key != key:
            self._check_planes((Y, U, V))
            self._args = _plane_args((Y, U, V), True)
            self._args_key = key
        ptrs, pitch, fstride = self._args
        F = Y.shape[0] if Y.dim() == 3 else 1
        dev = Y.device
        if out is None:
            out = torch.empty((max(F - n_halo, 0), 8), dtype=torch.float64, device=dev)
        elif (out.dtype != torch.float64 or out.device != dev or not out.is_contiguous()
              or out.numel() < 8 * max(F - n_halo, 0)):
            raise ValueError("out must be a contiguous float64 tensor of at least [n_frames - n_halo, 8] on %s" % dev)
        need = self._scratch_need.get(F)
        if need is None:
            need = self._scratch_need[F] = self.scratch_bytes(F)
        if scratch is None:
            if self._scratch is None or self._scratch.numel() < need // 8 + 1 or self._scratch.device != dev:
                self._scratch = torch.empty(need // 8 + 1, dtype=torch.float64, device=dev)
            scratch = self._scratch
        st = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
        _check(self._L.vca_analyze(self._h, ptrs, pitch, fstride, F, n_halo, scratch.data_ptr(),
                                   scratch.numel() * scratch.element_size(), out.data_ptr(), st),
               "vca_analyze")
        return out

    def analyze_host(self, Y, U, V, n_halo: int = 0, chunk_frames: int = 8, stream=None) -> np.ndarray:
        """Host planes (torch CPU tensors, ideally pinned) -> structured numpy records."""
        import torch

        self._check_planes((Y, U, V))
        ptrs, pitch, fstride = _plane_args((Y, U, V), False)
        F = Y.shape[0] if Y.dim() == 3 else 1
        out = np.zeros(max(F - n_halo, 0), dtype=RECORD_DTYPE)
        st = stream if stream is not None else torch.cuda.current_stream()
        _check(self._L.vca_analyze_host(self._h, ptrs, pitch, fstride, F, n_halo, chunk_frames,
                                        out.ctypes.data, st.cuda_stream), "vca_analyze_host")
        return out

    def profile_enable(self, on: bool = True):
        _check(self._L.vca_profile_enable(self._h, int(bool(on))), "vca_profile_enable")

    def profile_read(self):
        a, b, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(self._L.vca_profile_read(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)),
               "vca_profile_read")
        return a.value, b.value, n.value

    def debug_analyze(self, Y, U, V, n_halo: int = 0, scratch=None, stream=None):
        """TEST-ONLY: analyze() through the DUMP kernel instantiation.  Returns (records [F - n_halo, 8],
        scratch, per plane {"chk", "sumx", "H"} device tensors [F, count[p]])."""
        import torch

        self._check_planes((Y, U, V))
        ptrs, pitch, fstride = _plane_args((Y, U, V), True)
        F = Y.shape[0] if Y.dim() == 3 else 1
        dev = Y.device
        out = torch.empty((max(F - n_halo, 0), 8), dtype=torch.float64, device=dev)
        if scratch is None:
            scratch = torch.empty(self.scratch_bytes(F) // 8 + 1, dtype=torch.float64, device=dev)
        planes = []
        for p in range(3):
            C = self.info["count"][p]
            planes.append({"chk": torch.empty((F, C), dtype=torch.int64, device=dev),
                           "sumx": torch.empty((F, C), dtype=torch.int64, device=dev),
                           "H": torch.empty((F, C), dtype=torch.float64, device=dev)})
        P3 = ctypes.c_void_p * 3
        st = (stream if stream is not None else torch.cuda.current_stream(dev)).cuda_stream
        _check(self._L.vca_debug_analyze(self._h, ptrs, pitch, fstride, F, n_halo, scratch.data_ptr(),
                                         scratch.numel() * scratch.element_size(), out.data_ptr(),
                                         P3(*[d["chk"].data_ptr() for d in planes]),
                                         P3(*[d["sumx"].data_ptr() for d in planes]),
                                         P3(*[d["H"].data_ptr() for d in planes]), st), "vca_debug_analyze")
        return out, scratch, planes

    def debug_dump(self, Y, U, V):
        """TEST-ONLY: coefficients / sums / H / L of every block of one frame (device planes)."""
        self._check_planes((Y, U, V))
        ptrs, pitch, _ = _plane_args((Y, U, V), True)
        res = []
        cptr, sptr, hptr, lptr = [], [], [], []
        for p in range(3):
            C, n = self.info["count"][p], self.info["n"][p]
            d = {"coeffs": np.zeros((C, n, n), np.int32), "sumx": np.zeros(C, np.int64),
                 "H": np.zeros(C, np.float64), "L": np.zeros(C, np.float64)}
            res.append(d)
            cptr.append(d["coeffs"].ctypes.data)
            sptr.append(d["sumx"].ctypes.data)
            hptr.append(d["H"].ctypes.data)
            lptr.append(d["L"].ctypes.data)
        P3 = ctypes.c_void_p * 3
        _check(self._L.vca_debug_dump(self._h, ptrs, pitch, P3(*cptr), P3(*sptr), P3(*hptr), P3(*lptr)),
               "vca_debug_dump")
        return res


def version() -> str:
    return lib().vca_version().decode()


def status_string(code: int) -> str:
    return lib().vca_status_string(code).decode()
