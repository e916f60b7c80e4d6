"""Suite self-test driver (run by tests/test_mutation_gpu.py in a subprocess with VCA_LIB set to a
-DVCA_MUTATE build of libvca): for configs 3 and 4 at full UHD size, add 1 to ONE coefficient
of one block of one plane -- in the production kernel instantiation, the DUMP instantiation, or
both (vca_debug_mutate) -- and run the parity suite's own checks (tests/parity_util.py) on two
frames.  Prints one JSON object: per case, which checks went red.  A case with the mutation off
is the control and must stay green."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import torch  # noqa: E402

from paper_2304_12384_b200 import synth, vca  # noqa: E402
from parity_util import Pair, assert_checks, assert_records, oracle_checks  # noqa: E402


def verdict(pair, planes, cpu):
    """Run the suite's checks; return the list of those that failed."""
    red = []
    rec, hy, ch, recd, hyd, same = pair.analyze(*planes, strict=False)
    if not same:
        red.append("production_vs_dump_bitwise")
    r, rhy, rch = cpu
    try:
        assert_checks(ch, rch)
    except AssertionError:
        red.append("integer_checks_vs_oracle")
    try:
        assert_records(rec, r, rtol=1e-12)
    except AssertionError:
        red.append("records_vs_oracle_1e-12")
    return red


def main():
    L = vca.lib()
    out = {"lib": os.environ.get("VCA_LIB"), "cases": []}
    for cfg in (3, 4):
        c = synth.CONFIGS[cfg]
        Y, U, V = synth.config_frames(cfg, device="cuda", n_frames=2)
        cpu = oracle_checks(Y, U, V, c.bit_depth, c.block_size, c.lowpass)
        pair = Pair(c.width, c.height, c.bit_depth, c.block_size, c.lowpass)
        assert L.vca_debug_mutate(-1, -1, -1, 0) == 0, "not a VCA_MUTATE build"
        pair.reset(0)
        out["cases"].append({"cfg": cfg, "control": True, "red": verdict(pair, (Y, U, V), cpu)})
        for plane in range(3):
            C, n = pair.info["count"][plane], pair.info["n"][plane]
            for blk in (C + C // 2 + 3, 2 * C - 1):        # frame 1: a middle block, the last block
                for which in (1, 2, 3):                     # production, DUMP, both
                    pos = n + 2                              # (i, j) = (1, 2)
                    assert L.vca_debug_mutate(plane, blk, pos, which) == 0
                    pair.reset(0)
                    red = verdict(pair, (Y, U, V), cpu)
                    out["cases"].append({"cfg": cfg, "plane": plane, "block": int(blk), "pos": pos,
                                         "which": which, "red": red})
        L.vca_debug_mutate(-1, -1, -1, 0)
        del Y, U, V, pair
    print(json.dumps(out))


if __name__ == "__main__":
    main()
