"""B200-native hot path of VCA v2.0 (arxiv 2304.12384): blockwise integer-DCT
energy features E_Y, h, L_Y, E_U, L_U, E_V, L_V on sm_100a.

The compute lives in ``libvca.so`` (CUDA, C ABI in ``include/vca.h``);
``vca`` is its ctypes binding and ``synth`` the seeded input generators.
"""
from .vca import FEATURES, RECORD_DTYPE, Analyzer, VcaError, lib, records_to_numpy, status_string, version  # noqa: F401

__all__ = ["Analyzer", "VcaError", "FEATURES", "RECORD_DTYPE", "records_to_numpy", "lib", "version",
           "status_string"]
