"""How far inside the 1e-6 parity bar the CUDA path sits: the largest relative difference per
feature against the oracle on the first 120 frames of configs 1-4 (printed with -s; the
numbers in profiles/r01e/parity_margins.txt come from this test).  The two sides differ only
in FP64 summation order, so every feature must agree to 1e-12."""
import numpy as np
import pytest

import oracle
from paper_2304_12384_b200 import Analyzer, records_to_numpy, synth

pytestmark = pytest.mark.gpu

FEATS = ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V")


@pytest.mark.parametrize("cfg", (1, 2, 3, 4))
def test_parity_margins(cfg):
    c = synth.CONFIGS[cfg]
    F = min(c.n_frames, 120)
    Y, U, V = synth.with_pitch(synth.config_frames(cfg, device="cuda", n_frames=F))
    a = Analyzer(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
    g = records_to_numpy(a.analyze(Y, U, V))
    r = oracle.analyze(*synth.as_numpy_planes(Y, U, V), c.bit_depth, c.block_size, c.lowpass)
    worst = {}
    for f in FEATS:
        nz = r[f] != 0.0
        assert np.all(g[f][~nz] == 0.0), f
        rel = np.abs(g[f][nz] - r[f][nz]) / np.abs(r[f][nz])
        worst[f] = float(rel.max()) if rel.size else 0.0
    print("config %d: %s" % (cfg, "  ".join("%s %.2e" % kv for kv in worst.items())))
    assert max(worst.values()) <= 1e-12, worst
