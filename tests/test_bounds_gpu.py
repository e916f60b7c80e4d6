"""Debug-build check (compute-sanitizer is unavailable on this pool): the kernels rebuilt
with VCA_DEBUG_BOUNDS -- every data-path shared-memory access bounds- and alignment-checked
against the dynamic shared-memory size, every per-block H_Y store index-checked, a trap on
violation -- run the small-geometry parity cases (all kernel families, ragged strips,
partial blocks, extremes) in a subprocess and must still match the oracle."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_parity_under_bounds_checks(tmp_path):
    from paper_2304_12384_b200 import build

    lib = build.build(force=True, out=str(tmp_path / "libvca_bounds.so"), defines=("VCA_DEBUG_BOUNDS",))
    env = dict(os.environ, VCA_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_parity_gpu.py"), "-k",
                        "parity_small or extreme or clamp or golden or split or analyze_host"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "VCA_DEBUG_BOUNDS" not in r.stdout + r.stderr
