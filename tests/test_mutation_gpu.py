"""The parity suite's self-test (VERDICT r01 "make the production kernel's integers observable,
then prove the suite catches one wrong coefficient"): a -DVCA_MUTATE build of libvca adds 1 to
one AC coefficient of one block of the Y, U or V plane of configs 3 and 4 (full UHD size), in
the production kernel instantiation, the DUMP one, or both; the suite's checks must go red in
every case and stay green with the mutation off."""
import json
import os
import subprocess
import sys

import pytest

from paper_2304_12384_b200 import build

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def mutation_lib():
    out = os.path.join(build.HERE, "variants", "libvca_mutate.so")
    if not os.path.exists(out) or any(os.path.getmtime(s) > os.path.getmtime(out) for s in build.sources()):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        build.build(force=True, out=out, defines=["VCA_MUTATE"])
    return out


def test_suite_catches_one_wrong_coefficient():
    env = dict(os.environ, VCA_LIB=mutation_lib())
    res = subprocess.run([sys.executable, os.path.join(HERE, "mutation_probe.py")], capture_output=True, text=True,
                         env=env, timeout=1200)
    assert res.returncode == 0, res.stderr[-4000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    cases = out["cases"]
    assert len(cases) == 2 * (1 + 3 * 2 * 3)
    for c in cases:
        if c.get("control"):
            assert c["red"] == [], c                      # no mutation: the suite is green
            continue
        assert c["red"], c                                # every single-coefficient error is caught
        if c["which"] == 1:                               # production kernel only
            assert "production_vs_dump_bitwise" in c["red"], c
        else:                                             # DUMP kernel (alone or with production)
            assert "integer_checks_vs_oracle" in c["red"], c
