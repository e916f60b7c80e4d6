#!/usr/bin/env python
"""Writes tests/golden/derived.json: expected values that follow from the definitions
alone -- plain math (math.cos/exp/sqrt, Python ints, math.fsum), no oracle/ and no CUDA.

* basis fingerprints of T_n = round(64 sqrt(2) c_k cos(pi (2x+1) k / 2n)) (R-1)
* the 8x8 checkerboard texture energy of S:197-199 under R-1/R-2 by O(n^4) brute force
* the frame-level closed-form fixture of SURVEY.md §8(c) C3: E_Y = w* a / n,
  h = w* |a1 - a0| / n, L = sqrt(v n), w* = exp(15/16) = w_n(n/2, n/2) for every n

usage: python tests/golden/make_golden.py   (rewrites derived.json next to this file)
"""
import json
import math
import os


def basis(n):
    return [[int(round(64.0 * math.sqrt(2.0) * (1 / math.sqrt(2.0) if k == 0 else 1.0)
                       * math.cos(math.pi * (2 * x + 1) * k / (2 * n)))) for x in range(n)] for k in range(n)]


def checkerboard_H():
    n = 8
    T = basis(n)
    X = [[255 * ((x + y) % 2) for x in range(n)] for y in range(n)]
    C = [[sum(T[i][y] * T[j][x] * X[y][x] for y in range(n) for x in range(n)) for j in range(n)] for i in range(n)]
    return math.fsum(math.exp(abs((i * j / (n * n)) ** 2 - 1.0)) * abs(C[i][j]) / (4096.0 * n)
                     for i in range(n) for j in range(n) if (i, j) != (0, 0))


def main():
    out = {"_doc": __doc__.strip().splitlines()[0] + " Regenerate with make_golden.py."}
    out["basis"] = {str(n): {"cite": "R-1 (P:58; S:151, S:163); SURVEY.md 8(c) C3 fingerprints",
                             "sum_abs": sum(abs(v) for r in basis(n) for v in r),
                             "sum_sq": sum(v * v for r in basis(n) for v in r),
                             "row1": basis(n)[1]} for n in (4, 8, 16, 32)}
    out["checkerboard_8x8_H"] = {"cite": "S:197-199 (brute-force regression constant), R-1, R-2",
                                 "value": checkerboard_H()}
    ws = math.exp(15.0 / 16.0)
    frames = {}
    for lowpass, n, nc in ((False, 32, 16), (True, 16, 8)):
        frames["lowpass" if lowpass else "full"] = {
            "cite": "SURVEY.md 8(c) C3 frame-level closed form; S:233-234",
            "setup": "luma 128x64, w = 32, each luma block 128 + a s(x)s(y), s = T_n[n/2]/64 "
                     "(2x2-upsampled on the n = 16 grid in low-pass); U = 100, V = 200; frame A a = 50, frame B a = 20",
            "n": n, "n_c": nc,
            "E_Y": [ws * 50 / n, ws * 20 / n], "h": [0.0, ws * 30 / n],
            "L_Y": math.sqrt(128 * n), "E_U": 0.0, "E_V": 0.0,
            "L_U": math.sqrt(100 * nc), "L_V": math.sqrt(200 * nc)}
    out["closed_form_frames"] = frames
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "derived.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(path)


if __name__ == "__main__":
    main()
