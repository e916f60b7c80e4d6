"""Shared helpers of the GPU parity tests: the CUDA path (through the C ABI) against the CPU
oracle on the same seeded bytes, and the production kernel instantiation against the DUMP
instantiation bit for bit.

Bar (BASELINE.json north star; R-11): integer DCT coefficients, DC sums and the
per-block AC checksums bit-exact; per-frame features within 1e-6 relative (and, as a tighter
self-imposed check, 1e-12: the two sides differ only in FP64 summation order), an exact 0
reproduced as exactly 0.  Production vs DUMP instantiation: records and per-block H_Y
identical bit for bit -- one wrong coefficient in either moves a record by >= w_min / (4096 n)
/ (C n^2) absolute, thousands of ulps, so this ties the production kernel's integers to the
DUMP kernel's, which the checksums pin to the oracle.
"""
import numpy as np
import torch

import oracle
from paper_2304_12384_b200 import Analyzer, records_to_numpy, synth

RTOL = 1e-6
FEATS = ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V")


def assert_records(gpu, ref, rtol=RTOL):
    assert len(gpu) == len(ref)
    assert np.array_equal(gpu["poc"], ref["poc"])
    for f in FEATS:
        g, r = gpu[f], ref[f]
        zero = r == 0.0
        assert np.all(g[zero] == 0.0), f
        rel = np.abs(g[~zero] - r[~zero]) / np.abs(r[~zero])
        assert rel.size == 0 or rel.max() <= rtol, (f, float(rel.max()))


def planes_cuda(Y, U, V):
    """Device copies with 16-byte-aligned row pitch (libvca contract)."""
    return synth.with_pitch(tuple(p.cuda() for p in (Y, U, V)))


class Pair:
    """Two contexts of one geometry fed the same call sequence: `prod` through vca_analyze
    (the production kernel instantiation), `dbg` through vca_debug_analyze (the DUMP
    instantiation with the per-block integer outputs)."""

    def __init__(self, W, H, bd, w, lp):
        self.prod = Analyzer(W, H, bd, w, lp)
        self.dbg = Analyzer(W, H, bd, w, lp)
        self.info = self.prod.info

    def reset(self, poc=0):
        self.prod.reset(poc)
        self.dbg.reset(poc)

    def analyze(self, Y, U, V, n_halo=0, strict=True):
        """-> (records, H_Y [F][C_Y], per-plane {"chk", "sumx", "H"} numpy [F][C_p]), after
        asserting that both instantiations agree bit for bit on records and H_Y.  With
        strict=False: -> (production records, production H_Y, DUMP checks, DUMP records, DUMP
        H_Y, identical) without asserting."""
        F = Y.shape[0]
        CY = self.info["count"][0]
        sp = torch.empty(self.prod.scratch_bytes(F) // 8 + 1, dtype=torch.float64, device=Y.device)
        rp = self.prod.analyze(Y, U, V, n_halo=n_halo, scratch=sp)
        rd, sd, checks = self.dbg.debug_analyze(Y, U, V, n_halo=n_halo)
        torch.cuda.synchronize()
        rec, recd = records_to_numpy(rp), records_to_numpy(rd)
        hy, hyd = sp[:F * CY], sd[:F * CY]
        same_rec, same_hy = rec.tobytes() == recd.tobytes(), torch.equal(hy, hyd)
        ch = [{k: v.cpu().numpy() for k, v in d.items()} for d in checks]
        hy = hy.view(F, CY).cpu().numpy()
        if not strict:
            return rec, hy, ch, recd, hyd.view(F, CY).cpu().numpy(), same_rec and same_hy
        assert same_rec, "production and DUMP records differ"
        assert same_hy, "production and DUMP per-block H_Y differ"
        return rec, hy, ch


def assert_checks(got, want, frames=None):
    """Per-block integer checks bit-exact (AC checksum, sample sum) and H within 1e-12, every
    plane; `frames` selects rows of `got` matching `want`."""
    for p in range(3):
        g = {k: (v if frames is None else v[frames]) for k, v in got[p].items()}
        w = want[p]
        assert g["chk"].shape == w["chk"].shape, p
        bad = np.argwhere(g["chk"] != w["chk"])
        assert bad.size == 0, ("AC checksum differs", p, bad[:5].tolist())
        bad = np.argwhere(g["sumx"] != w["sumx"])
        assert bad.size == 0, ("sample sum differs", p, bad[:5].tolist())
        ref = w["H"]
        assert np.all(np.abs(g["H"] - ref) <= 1e-12 * np.maximum(ref, 1e-300)), ("H", p)


def oracle_checks(Y, U, V, bd, w, lp, n_halo=0, first_poc=0, prev_HY=None):
    """Oracle records, H_Y and per-block checks of host copies of the planes."""
    npl = synth.as_numpy_planes(Y, U, V)
    return oracle.analyze(*npl, bd, w, lp, n_halo=n_halo, first_poc=first_poc, prev_HY=prev_HY, want_HY=True,
                          want_checks=True)
