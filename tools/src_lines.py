#!/usr/bin/env python
"""Attribute ncu SASS-level stall samples (--page source --csv --print-source sass) to CUDA
source lines using nvdisasm --print-line-info on the kernel's cubin.
usage: src_lines.py SOURCE_SASS.csv CUBIN MANGLED_KERNEL_NAME [--top 40]"""
import argparse
import collections
import csv
import re
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("cubin")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    dis = subprocess.run(["nvdisasm", "--print-line-info", a.cubin], capture_output=True, text=True).stdout
    line_of = {}
    cur = None
    infn = False
    for l in dis.splitlines():
        if l.startswith(".text.") or "\t.text." in l or l.strip().startswith(".section\t.text."):
            infn = a.kernel in l
            cur = None
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = "%s:%s" % (m.group(1).split("/")[-1], m.group(2))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(a.csv)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0][ix["Address"]], 16)
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(float(r[ix[key]] or 0) for r in data)
    agg = collections.Counter()
    inst = collections.Counter()
    for r in data:
        off = int(r[ix["Address"]], 16) - base
        ln = line_of.get(off, "?")
        agg[ln] += float(r[ix[key]] or 0)
        inst[ln] += float(r[ix["Instructions Executed"]] or 0)
    for ln, v in agg.most_common(a.top):
        print("%5.2f %%  inst %11d  %s" % (100 * v / tot, inst[ln], ln))


if __name__ == "__main__":
    main()
