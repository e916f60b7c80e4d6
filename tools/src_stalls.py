#!/usr/bin/env python
"""Aggregate an ncu source page (--page source --csv --print-source sass) of one kernel:
stall samples by opcode and by stall reason, and the hottest instructions.
usage: src_stalls.py SOURCE.csv [--top 40]"""
import argparse
import collections
import csv
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
    tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    by_op = collections.Counter()
    by_reason = collections.Counter()
    by_op_reason = collections.defaultdict(collections.Counter)
    inst = collections.Counter()
    for r in data:
        src = r[ix["Source"]].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", src)
        op = m.group(2) if m else src
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        by_op[op] += s
        inst[op] += float(r[ix["Instructions Executed"]] or 0)
        for h in reasons:
            v = float(r[ix[h]] or 0)
            by_reason[h] += v
            by_op_reason[op][h] += v
    print("total stall samples: %d" % tot)
    print("\n## by reason")
    for k, v in by_reason.most_common():
        if v:
            print("%-24s %6.1f %%" % (k, 100 * v / tot))
    print("\n## by opcode (share of samples, executed warp-instructions, top reasons)")
    for k, v in by_op.most_common(a.top):
        top = ", ".join("%s %.0f%%" % (h[6:], 100 * c / v) for h, c in by_op_reason[k].most_common(3) if c)
        print("%-28s %6.1f %%  inst %10d  | %s" % (k, 100 * v / tot, inst[k], top))
    print("\n## hottest instructions")
    data.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    for r in data[:a.top]:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        top = sorted(((float(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]
        print("%5.2f %%  %s  %-60s  %s" % (100 * s / tot, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:60],
                                          ", ".join("%s %d" % (n, v) for v, n in top if v)))


if __name__ == "__main__":
    main()
