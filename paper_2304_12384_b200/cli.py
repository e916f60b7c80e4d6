"""Command-line entry point (SPEC.md cli S:471-508).

    python -m paper_2304_12384_b200.cli analyze INPUT [-o OUT.csv] [options]
    python -m paper_2304_12384_b200.cli bench   INPUT [options]

INPUT is a .y4m file (or '-' for a Y4M pipe) or a headerless .yuv/.raw file with
--width/--height (and --bit-depth, --chroma).  `analyze` streams the whole input
through the GPU (native reader thread + pinned batches + overlapped H2D,
vca_analyze_stream) and writes the features CSV (POC,E_Y,h,L_Y,E_U,L_U,E_V,L_V,
6 decimals) to OUT or standard output, with the per-feature mean/max
summary on standard error.  `bench` runs the same analysis without writing a
CSV and prints `frames=<n> seconds=<s> fps=<f>`.

Exit codes: 0 success, 1 usage error, 2 input error.
The SI/TI mode of SPEC's CPU program is not part of this build.
"""
from __future__ import annotations

import argparse
import os
import sys

from .vca import Analyzer, VcaError
from . import vcaio


class _Usage(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _Usage(message)


def _parser():
    ap = _Parser(prog="python -m paper_2304_12384_b200.cli", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd")
    for name in ("analyze", "bench"):
        p = sub.add_parser(name)
        p.add_argument("input")
        if name == "analyze":
            p.add_argument("-o", "--output", default="-")
        p.add_argument("--format", choices=("y4m", "raw"), default=None,
                       help="input format (default: from the extension; '-' is Y4M)")
        p.add_argument("--width", type=int, default=0)
        p.add_argument("--height", type=int, default=0)
        p.add_argument("--bit-depth", type=int, default=8, choices=(8, 10))
        p.add_argument("--chroma", type=int, default=420, choices=(420, 422, 444))
        p.add_argument("--block-size", type=int, default=0, choices=(0, 4, 8, 16, 32),
                       help="luma block size (0 = auto: 32 if H >= 2160, 16 if >= 1080, else 8)")
        p.add_argument("--low-pass", action="store_true", help="low-pass DCT (P:60)")
        p.add_argument("--batch-frames", type=int, default=32)
        p.add_argument("--device", type=int, default=0)
    return ap


def run(argv=None) -> int:
    try:
        args = _parser().parse_args(argv)
        if args.cmd is None:
            raise _Usage("missing subcommand (analyze | bench)")
        fmt = args.format
        if fmt is None:
            ext = os.path.splitext(args.input)[1].lower()
            fmt = "y4m" if (args.input == "-" or ext == ".y4m") else "raw" if ext in (".yuv", ".raw") else None
            if fmt is None:
                raise _Usage("cannot infer the input format from %r; pass --format" % args.input)
        if fmt == "raw" and (args.width <= 0 or args.height <= 0):
            raise _Usage("raw input needs --width and --height")
    except _Usage as e:
        sys.stderr.write("usage error: %s\n" % e)
        return 1
    try:
        reader = vcaio.Reader(args.input, fmt, args.width, args.height, args.bit_depth, args.chroma)
        import torch

        if torch.cuda.is_available():
            torch.cuda.set_device(args.device)
        info = reader.info
        if reader.warnings & vcaio.WARN_TRAILING_BYTES:
            sys.stderr.write("warning: trailing partial frame discarded\n")
        if reader.warnings & vcaio.WARN_X_TOKENS:
            sys.stderr.write("warning: Y4M X tokens ignored\n")
        an = Analyzer(info["width"], info["height"], info["bit_depth"], args.block_size, args.low_pass,
                      info["chroma"])
        rec, seconds = vcaio.analyze_stream(an, reader, args.batch_frames)
        n = len(rec)
        if n == 0:
            raise VcaError(-1, "empty stream")  # EmptyStream
        if args.cmd == "bench":
            sys.stdout.write("frames=%d seconds=%.6f fps=%.2f\n" % (n, seconds, n / seconds if seconds > 0 else 0.0))
            return 0
        vcaio.write_csv(args.output, rec)
        mean, mx = vcaio.summarize(rec)
        sys.stderr.write("# frames=%d seconds=%.6f fps=%.2f\n" % (n, seconds, n / seconds if seconds > 0 else 0.0))
        sys.stderr.write("# mean " + " ".join("%s=%.6f" % kv for kv in mean.items()) + "\n")
        sys.stderr.write("# max  " + " ".join("%s=%.6f" % kv for kv in mx.items()) + "\n")
        return 0
    except VcaError as e:
        sys.stderr.write("input error: %s\n" % e)
        return 2


def main():
    sys.exit(run())


if __name__ == "__main__":
    main()
