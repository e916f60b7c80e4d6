"""Pins for the CPU oracle (oracle/vca_oracle.c) against what the paper,
SPEC.md and mathematics fix -- never against the oracle itself.

Each test names the passage (P:n = PAPER.md line, S:n = SPEC.md line) or
the DESIGN.md reading (R-k) it pins.  Independent machinery used here:
scipy's orthonormal DCT-II (library routine), exact Python-integer
brute force O(n^4), numpy edge padding, closed forms, math.fsum.
"""
import math

import numpy as np
import pytest
from scipy.fft import dct, dctn

pytestmark = []

SIZES = (4, 8, 16, 32)
WSTAR = math.exp(15.0 / 16.0)  # w_n(n/2, n/2) = exp(|(1/4)^2 - 1|) for every n


def ortho_basis(n):
    """Orthonormal DCT-II matrix Phi (rows = frequencies) from scipy."""
    return dct(np.eye(n), type=2, norm="ortho", axis=0)


def brute_coeffs(T, X):
    """Exact C_ij = sum_y sum_x T[i][y] T[j][x] X[y][x] with Python ints, O(n^4)."""
    n = len(X)
    T = [[int(v) for v in row] for row in T]
    X = [[int(v) for v in row] for row in X]
    return [[sum(T[i][y] * T[j][x] * X[y][x] for y in range(n) for x in range(n)) for j in range(n)]
            for i in range(n)]


def brute_H(C, n):
    """S:194 with R-2 scaling, weights via math.exp, exact-ish sum via fsum."""
    terms = []
    for i in range(n):
        for j in range(n):
            if (i, j) == (0, 0):
                continue
            terms.append(math.exp(abs((i * j / (n * n)) ** 2 - 1.0)) * abs(C[i][j]) / (4096.0 * n))
    return math.fsum(terms)


# --------------------------------------------------------------------- basis (R-1)

@pytest.mark.parametrize("n", SIZES)
def test_basis_is_rounded_scaled_dct2(oracle_mod, n):
    """R-1: T_n = round(64 sqrt(n) Phi_n) elementwise (scipy's orthonormal DCT-II)."""
    T = oracle_mod.basis(n).astype(np.float64)
    R = 64.0 * math.sqrt(n) * ortho_basis(n)
    assert np.all(np.abs(T - R) <= 0.5)
    assert np.array_equal(T, np.rint(R))


@pytest.mark.parametrize("n", SIZES)
def test_basis_structure(oracle_mod, n):
    T = oracle_mod.basis(n).astype(np.int64)
    assert np.all(T[0] == 64)                                   # DC row
    assert np.all(T[1:].sum(axis=1) == 0)                       # AC rows sum to zero
    for k in range(n):
        sym = T[k] == T[k][::-1]
        anti = T[k] == -T[k][::-1]
        assert (sym.all() if k % 2 == 0 else anti.all())        # even symmetric, odd antisymmetric
    assert np.all(np.abs(T) <= 90)                              # fits int8 (tensor-core operand)
    if n > 4:                                                   # nesting: T_n[2m][x<n/2] = T_{n/2}[m][x]
        Th = oracle_mod.basis(n // 2).astype(np.int64)
        assert np.array_equal(T[0::2, : n // 2], Th)
    # T[n/2] is exactly +-64: the single-coefficient closed form below relies on it
    assert np.all(np.abs(T[n // 2]) == 64)


# --------------------------------------------------------------------- integer DCT (R-1)

@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("bd", (8, 10))
def test_dct_exact_brute_force(oracle_mod, n, bd):
    """The oracle's separable product equals the O(n^4) definition exactly."""
    rng = np.random.default_rng(100 + n + bd)
    T = oracle_mod.basis(n)
    hi = (1 << bd) - 1
    for trial in range(2 if n == 32 else 4):
        X = rng.integers(0, hi + 1, size=(n, n))
        plane = X.astype(np.uint8 if bd == 8 else np.uint16)
        C, sumx, H, L = oracle_mod.block(plane, bd, n, False, 0, 0)
        Cb = brute_coeffs(T, X)
        assert [[int(v) for v in row] for row in C] == Cb
        assert sumx == int(X.sum())
        assert C[0][0] == 4096 * sumx


@pytest.mark.parametrize("n", SIZES)
def test_dct_close_to_float_dct2(oracle_mod, n):
    """C/(4096 n) differs from scipy's orthonormal DCT-II only by the basis
    rounding: |E| <= (|dT| X |T|^T + |R| X |dT|^T)/(4096 n) elementwise."""
    rng = np.random.default_rng(7 + n)
    T = oracle_mod.basis(n).astype(np.float64)
    R = 64.0 * math.sqrt(n) * ortho_basis(n)
    dT = np.abs(T - R)
    for _ in range(3):
        X = rng.integers(0, 256, size=(n, n)).astype(np.float64)
        C, _, _, _ = oracle_mod.block(X.astype(np.uint8), 8, n, False, 0, 0)
        got = C.astype(np.float64) / (4096.0 * n)
        ref = dctn(X, type=2, norm="ortho")
        bound = (dT @ X @ np.abs(T).T + np.abs(R) @ X @ dT.T) / (4096.0 * n)
        assert np.all(np.abs(got - ref) <= bound + 1e-9)
        # DC is exact: sum(X)/n
        assert got[0, 0] == X.sum() / n


def test_spec_dct_examples(oracle_mod):
    """constant 8x8 v=128 -> DC 1024, AC 0; impulse -> DC 0.125;
    rows identical -> C[i>0][.] = 0."""
    C, _, H, L = oracle_mod.block(np.full((8, 8), 128, np.uint8), 8, 8, False, 0, 0)
    assert C[0, 0] / (4096 * 8) == 1024.0 and np.all(C.ravel()[1:] == 0) and H == 0.0
    imp = np.zeros((8, 8), np.uint8)
    imp[0, 0] = 1
    C, _, _, _ = oracle_mod.block(imp, 8, 8, False, 0, 0)
    assert C[0, 0] / (4096 * 8) == 0.125
    rows = np.tile(np.arange(8, dtype=np.uint8) * 30, (8, 1))
    C, _, _, _ = oracle_mod.block(rows, 8, 8, False, 0, 0)
    assert np.all(C[1:, :] == 0) and np.any(C[0, 1:] != 0)


@pytest.mark.parametrize("n", SIZES)
def test_single_coefficient_closed_form(oracle_mod, n):
    """X = c + a s(x)s(y) with s = T_n[n/2]/64 (a +-1 pattern) has exactly
    C_00 = (64 n)^2 c, C[n/2][n/2] = (64 n)^2 a and nothing else; so
    H = w_n(n/2, n/2) |a| n (north star: 'a single-coefficient basis-pattern
    block gives energy in that coefficient only')."""
    T = oracle_mod.basis(n).astype(np.int64)
    s = T[n // 2] // 64
    for c, a in ((128, 50), (100, -37), (30, 25)):
        X = (c + a * np.outer(s, s)).astype(np.uint8)
        C, sumx, H, L = oracle_mod.block(X, 8, n, False, 0, 0)
        want = np.zeros((n, n), np.int64)
        want[0, 0] = (64 * n) ** 2 * c
        want[n // 2, n // 2] = (64 * n) ** 2 * a
        assert np.array_equal(C, want)
        assert H == pytest.approx(WSTAR * abs(a) * n, rel=1e-14)
        assert L == math.sqrt(c * n)
        # s (x) 1 -> only coefficient (n/2, 0), weight e
        X2 = (c + a * np.outer(s, np.ones(n, np.int64))).astype(np.uint8)
        C2, _, H2, _ = oracle_mod.block(X2, 8, n, False, 0, 0)
        want2 = np.zeros((n, n), np.int64)
        want2[0, 0] = (64 * n) ** 2 * c
        want2[n // 2, 0] = (64 * n) ** 2 * a
        assert np.array_equal(C2, want2)
        assert H2 == pytest.approx(math.e * abs(a) * n, rel=1e-14)


@pytest.mark.parametrize("n", SIZES)
def test_linearity_and_offset(oracle_mod, n):
    """C(2X) = 2 C(X) exactly and H(2B) = 2 H(B) bit-exactly;
    S:238: adding an in-range constant changes only the DC term."""
    rng = np.random.default_rng(n)
    X = rng.integers(0, 120, size=(n, n))
    C1, _, H1, _ = oracle_mod.block(X.astype(np.uint8), 8, n, False, 0, 0)
    C2, _, H2, _ = oracle_mod.block((2 * X).astype(np.uint8), 8, n, False, 0, 0)
    C3, _, H3, _ = oracle_mod.block((X + 17).astype(np.uint8), 8, n, False, 0, 0)
    assert np.array_equal(C2, 2 * C1) and H2 == 2 * H1
    d = C3 - C1
    assert d[0, 0] == 4096 * n * n * 17 and np.all(d.ravel()[1:] == 0) and H3 == H1


@pytest.mark.parametrize("n", SIZES)
def test_parseval_loose(oracle_mod, n):
    """S:146 holds only approximately for the integer basis (<= 0.3 %)."""
    rng = np.random.default_rng(50 + n)
    X = rng.integers(0, 256, size=(n, n))
    C, _, _, _ = oracle_mod.block(X.astype(np.uint8), 8, n, False, 0, 0)
    e_c = float(((C.astype(np.float64) / (4096.0 * n)) ** 2).sum())
    e_x = float((X.astype(np.float64) ** 2).sum())
    assert abs(e_c / e_x - 1.0) < 3e-3


# --------------------------------------------------------------------- H and L

def test_checkerboard_H(oracle_mod):
    """8x8 checkerboard 0/255 pinned by an independent brute force
    (Python ints + fsum): 5641.094923288223 under R-1/R-2; within 0.05 % of
    SPEC's float reading (orthonormal float DCT, computed here with scipy)."""
    X = np.array([[255 * ((x + y) % 2) for x in range(8)] for y in range(8)])
    _, _, H, _ = oracle_mod.block(X.astype(np.uint8), 8, 8, False, 0, 0)
    Cb = brute_coeffs(oracle_mod.basis(8), X)
    assert H == pytest.approx(brute_H(Cb, 8), rel=1e-13)
    assert H == pytest.approx(5641.094923288223, rel=1e-13)
    Cf = dctn(X.astype(np.float64), type=2, norm="ortho")
    Hf = math.fsum(math.exp(abs((i * j / 64.0) ** 2 - 1)) * abs(Cf[i, j])
                   for i in range(8) for j in range(8) if (i, j) != (0, 0))
    assert abs(H / Hf - 1) < 5e-4


@pytest.mark.parametrize("n", SIZES)
def test_H_brute_force_random(oracle_mod, n):
    rng = np.random.default_rng(200 + n)
    X = rng.integers(0, 256, size=(n, n))
    C, _, H, _ = oracle_mod.block(X.astype(np.uint8), 8, n, False, 0, 0)
    assert H == pytest.approx(brute_H(C.tolist(), n), rel=1e-12)


def test_weights(oracle_mod):
    """w(i,j) = exp(|(ij/n^2)^2 - 1|); symmetric; w(0,j) = e."""
    for n in SIZES:
        for i in range(n):
            for j in range(n):
                assert oracle_mod.weight(n, i, j) == oracle_mod.weight(n, j, i)
            assert oracle_mod.weight(n, 0, i) == pytest.approx(math.e, rel=1e-15)
        assert oracle_mod.weight(n, n // 2, n // 2) == pytest.approx(WSTAR, rel=1e-15)


def test_spec_luminescence_examples(oracle_mod):
    """const 8x8 v=128 -> 32.0; zero -> 0; const 16x16 v=64 -> 32.0."""
    assert oracle_mod.block(np.full((8, 8), 128, np.uint8), 8, 8, False, 0, 0)[3] == 32.0
    assert oracle_mod.block(np.zeros((8, 8), np.uint8), 8, 8, False, 0, 0)[3] == 0.0
    assert oracle_mod.block(np.full((16, 16), 64, np.uint8), 8, 16, False, 0, 0)[3] == 32.0


# --------------------------------------------------------------------- low-pass (R-5)

def test_spec_downsample_examples(oracle_mod):
    """77 -> 77; [10,20;30,40] tiles -> 25; 0/255 checkerboard -> 128
    (127.5 rounds half away from zero).  Observed through the DCT of the
    downsampled block: constant => AC = 0, sum = v n^2."""
    cases = ((np.full((8, 8), 77), 77), (np.tile(np.array([[10, 20], [30, 40]]), (4, 4)), 25),
             (np.array([[255 * ((x + y) % 2) for x in range(8)] for y in range(8)]), 128))
    for X, v in cases:
        C, sumx, H, L = oracle_mod.block(X.astype(np.uint8), 8, 8, True, 0, 0)
        assert C.shape == (4, 4) and sumx == 16 * v and H == 0.0 and np.all(C.ravel()[1:] == 0)


@pytest.mark.parametrize("w", (8, 16, 32))
@pytest.mark.parametrize("bd", (8, 10))
def test_lowpass_matches_numpy_mean(oracle_mod, w, bd):
    """Low-pass block = (2x2 sum + 2) >> 2 of the padded block, then the
    (w/2)-point DCT (R-5), checked with numpy reshape-sum + brute force."""
    rng = np.random.default_rng(300 + w + bd)
    hi = (1 << bd) - 1
    X = rng.integers(0, hi + 1, size=(w, w))
    plane = X.astype(np.uint8 if bd == 8 else np.uint16)
    C, sumx, H, _ = oracle_mod.block(plane, bd, w, True, 0, 0)
    s = X.reshape(w // 2, 2, w // 2, 2).sum(axis=(1, 3))
    d = (s + 2) // 4
    n = w // 2
    if n <= 8:
        assert [[int(v) for v in r] for r in C] == brute_coeffs(oracle_mod.basis(n), d)
    else:
        T = oracle_mod.basis(n).astype(object)
        assert [[int(v) for v in r] for r in C] == (T.dot(d.astype(object)).dot(T.T)).tolist()
    assert sumx == int(d.sum())


def test_lowpass_offset_exact(oracle_mod):
    """(s + 4c + 2) >> 2 = ((s + 2) >> 2) + c: an offset changes only DC in low-pass too."""
    rng = np.random.default_rng(9)
    X = rng.integers(0, 200, size=(32, 32))
    C1, _, H1, _ = oracle_mod.block(X.astype(np.uint8), 8, 32, True, 0, 0)
    C2, _, H2, _ = oracle_mod.block((X + 40).astype(np.uint8), 8, 32, True, 0, 0)
    assert H1 == H2 and np.array_equal(C1.ravel()[1:], C2.ravel()[1:])


# --------------------------------------------------------------------- grid, replication, clamp

@pytest.mark.parametrize("lowpass", (False, True))
def test_edge_replication_matches_numpy_pad(oracle_mod, lowpass):
    """out-of-range coordinates clamp to the nearest sample; equals
    numpy.pad(mode='edge') of the plane."""
    rng = np.random.default_rng(11)
    plane = rng.integers(0, 256, size=(40, 72)).astype(np.uint8)
    padded = np.pad(plane, ((0, 24), (0, 24)), mode="edge")
    for r in range(2):
        for c in range(3):
            a = oracle_mod.block(plane, 8, 32, lowpass, r, c)
            b = oracle_mod.block(padded, 8, 32, lowpass, r, c)
            assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]


def test_ten_bit_clamp(oracle_mod):
    """10-bit container values above 1023 are clamped to 1023."""
    X = np.full((8, 8), 1023, np.uint16)
    X[3, 4] = 4000
    a = oracle_mod.block(X, 10, 8, False, 0, 0)
    assert a[2] == 0.0 and a[1] == 64 * 1023


def test_block_rules(oracle_mod):
    """S:250 auto block size, S:249 chroma block, S:175 block count."""
    assert oracle_mod.resolve_block(2160, 0) == 32
    assert oracle_mod.resolve_block(1080, 0) == 16
    assert oracle_mod.resolve_block(720, 0) == 8
    assert oracle_mod.chroma_block(32) == 16 and oracle_mod.chroma_block(8) == 4 and oracle_mod.chroma_block(4) == 4
    assert oracle_mod.block_count(3840, 2160, 32) == 120 * 68
    assert oracle_mod.block_count(1920, 1080, 32) == 60 * 34
    assert oracle_mod.block_count(1920, 1080, 16) == 120 * 68


# --------------------------------------------------------------------- frame level

def _fixture_frames(a_values, lowpass):
    """Survey section 8(c) C3 closed-form fixture: luma 128x64 of blocks
    128 + a s(x)s(y) (s = T_n[n/2]/64 = the +-1 pattern), U = 100, V = 200."""
    n = 16 if lowpass else 32
    x = np.arange(n)
    s = np.where(((x % 4) == 0) | ((x % 4) == 3), 1, -1)  # (+,-,-,+,...) = sign cos(pi(2x+1)/4)
    blk = np.outer(s, s)
    if lowpass:
        blk = np.kron(blk, np.ones((2, 2), np.int64))      # 2x2-upsampled: downsample is exact
    Y = np.stack([np.tile(128 + a * blk, (2, 4)) for a in a_values]).astype(np.uint8)
    U = np.full((len(a_values), 32, 64), 100, np.uint8)
    V = np.full((len(a_values), 32, 64), 200, np.uint8)
    return Y, U, V


@pytest.mark.parametrize("lowpass", (False, True))
def test_frame_closed_form(oracle_mod, lowpass):
    """E_Y = w* a / n, h = w* |a1 - a0| / n, L_Y = sqrt(128 n), E_U = E_V = 0,
    L_U = sqrt(100 n_c), L_V = sqrt(200 n_c)  (w* = exp(15/16))."""
    Y, U, V = _fixture_frames((50, 20), lowpass)
    rec = oracle_mod.analyze(Y, U, V, 8, 32, lowpass)
    n, nc = (16, 8) if lowpass else (32, 16)
    assert rec["poc"].tolist() == [0, 1]
    assert rec["E_Y"][0] == pytest.approx(WSTAR * 50 / n, rel=1e-14)
    assert rec["E_Y"][1] == pytest.approx(WSTAR * 20 / n, rel=1e-14)
    assert rec["h"][0] == 0.0
    assert rec["h"][1] == pytest.approx(WSTAR * 30 / n, rel=1e-14)
    # means of equal irrational terms: exact up to summation rounding
    assert rec["L_Y"] == pytest.approx([math.sqrt(128 * n)] * 2, rel=1e-15)
    assert np.all(rec["E_U"] == 0.0) and np.all(rec["E_V"] == 0.0)
    assert rec["L_U"] == pytest.approx([math.sqrt(100 * nc)] * 2, rel=1e-15)
    assert rec["L_V"] == pytest.approx([math.sqrt(200 * nc)] * 2, rel=1e-15)
    if not lowpass:  # survey's printed values for the full case
        assert rec["E_Y"][0] == pytest.approx(3.9899835282233234, rel=1e-15)
        assert rec["h"][1] == pytest.approx(2.3939901169339937, rel=1e-15)


def _g(oracle_mod, seed=5, F=4, W=96, H=64, bd=8):
    from paper_2304_12384_b200 import synth
    return synth.as_numpy_planes(*synth.g_frames(seed, W, H, F, bd))


def test_constant_frame(oracle_mod):
    """constant frame -> E = 0, h = 0, L = sqrt(n v) (full and low-pass)."""
    for lowpass, n, nc in ((False, 32, 16), (True, 16, 8)):
        Y = np.full((2, 64, 96), 90, np.uint8)
        U = np.full((2, 32, 48), 60, np.uint8)
        V = np.full((2, 32, 48), 10, np.uint8)
        rec = oracle_mod.analyze(Y, U, V, 8, 32, lowpass)
        for f in ("E_Y", "E_U", "E_V", "h"):
            assert np.all(rec[f] == 0.0)
        assert rec["L_Y"] == pytest.approx([math.sqrt(n * 90)] * 2, rel=1e-15)
        assert rec["L_U"] == pytest.approx([math.sqrt(nc * 60)] * 2, rel=1e-15)


def test_recomposition_from_blocks(oracle_mod):
    """the frame features equal the per-block quantities averaged
    (fsum here, sequential in the oracle), h the SAD of H vectors."""
    Y, U, V = _g(oracle_mod, F=3, W=100, H=70)
    for lowpass in (False, True):
        w = 32
        rec, HY = oracle_mod.analyze(Y, U, V, 8, w, lowpass, want_HY=True)
        n = w // 2 if lowpass else w
        for t in range(3):
            for p, plane, wp, Ef, Lf in ((0, Y, w, "E_Y", "L_Y"), (1, U, 16, "E_U", "L_U"), (2, V, 16, "E_V", "L_V")):
                ph, pw = plane.shape[1:]
                rows, cols = -(-ph // wp), -(-pw // wp)
                Hs, Ls = [], []
                for r in range(rows):
                    for c in range(cols):
                        _, _, Hb, Lb = oracle_mod.block(plane[t], 8, wp, lowpass, r, c)
                        Hs.append(Hb)
                        Ls.append(Lb)
                npp = wp // 2 if lowpass else wp
                assert rec[Ef][t] == pytest.approx(math.fsum(Hs) / (len(Hs) * npp * npp), rel=1e-13)
                assert rec[Lf][t] == pytest.approx(math.fsum(Ls) / len(Ls), rel=1e-13)
                if p == 0:
                    assert np.array_equal(HY[t], np.array(Hs))
            if t > 0:
                want = math.fsum(abs(a - b) for a, b in zip(HY[t], HY[t - 1])) / (HY.shape[1] * n * n)
                assert rec["h"][t] == pytest.approx(want, rel=1e-13)


def test_h_properties(oracle_mod):
    """S:234 identical frames -> h = 0; S:239 symmetry; S:240 triangle inequality."""
    Y, U, V = _g(oracle_mod, seed=21, F=3)
    same = [np.stack([p[0], p[0]]) for p in (Y, U, V)]
    assert oracle_mod.analyze(*same, 8, 32, False)["h"][1] == 0.0
    A, B, C = 0, 1, 2
    def h(i, j):
        pl = [np.stack([p[i], p[j]]) for p in (Y, U, V)]
        return oracle_mod.analyze(*pl, 8, 32, False)["h"][1]
    assert h(A, B) == h(B, A)
    assert h(A, C) <= h(A, B) + h(B, C) + 1e-12


def test_noise_monotonicity(oracle_mod):
    """E_Y strictly increases over a 5-step noise-amplitude ladder."""
    rng = np.random.default_rng(3)
    base = 128.0
    noise = rng.standard_normal((64, 96))
    E = []
    for amp in (2, 4, 8, 16, 32):
        Y = np.clip(np.rint(base + amp * noise), 0, 255).astype(np.uint8)[None]
        U = np.full((1, 32, 48), 128, np.uint8)
        E.append(oracle_mod.analyze(Y, U, U, 8, 32, False)["E_Y"][0])
    assert all(b > a for a, b in zip(E, E[1:]))


def test_offset_invariance_frame(oracle_mod):
    """a constant offset leaves E_Y bit-identical (full and low-pass)."""
    Y, U, V = _g(oracle_mod, seed=8, F=2)
    Y = (Y // 2).astype(np.uint8)
    for lowpass in (False, True):
        a = oracle_mod.analyze(Y, U, V, 8, 32, lowpass)
        b = oracle_mod.analyze((Y + 50).astype(np.uint8), U, V, 8, 32, lowpass)
        assert np.array_equal(a["E_Y"], b["E_Y"]) and np.array_equal(a["h"], b["h"])


def test_halo_and_carry(oracle_mod):
    """splitting a sequence with a one-frame halo, or carrying
    the previous H vector, reproduces the unsplit records bit-exactly."""
    Y, U, V = _g(oracle_mod, seed=13, F=6)
    full, HY = oracle_mod.analyze(Y, U, V, 8, 32, True, want_HY=True)
    tail = oracle_mod.analyze(Y[2:], U[2:], V[2:], 8, 32, True, n_halo=1, first_poc=3)
    assert np.array_equal(tail, full[3:])
    tail2 = oracle_mod.analyze(Y[3:], U[3:], V[3:], 8, 32, True, prev_HY=HY[2], first_poc=3)
    assert np.array_equal(tail2, full[3:])


def test_thread_count_invariance(oracle_mod):
    """bit-identical for any thread count."""
    Y, U, V = _g(oracle_mod, seed=2, F=5)
    a = oracle_mod.analyze(Y, U, V, 8, 32, False, n_threads=1)
    b = oracle_mod.analyze(Y, U, V, 8, 32, False, n_threads=4)
    assert np.array_equal(a, b)


def test_first_frame_h_zero_and_nonneg(oracle_mod):
    """all values >= 0, h(poc 0) = 0."""
    Y, U, V = _g(oracle_mod, seed=4, F=3, bd=10)
    rec = oracle_mod.analyze(Y, U, V, 10, 16, False)
    assert rec["h"][0] == 0.0
    for f in ("E_Y", "h", "L_Y", "E_U", "L_U", "E_V", "L_V"):
        assert np.all(rec[f] >= 0)
    assert np.all(rec["h"][1:] > 0)


# --------------------------------------------------------------------- per-block integer checks

@pytest.mark.parametrize("W,H,bd,w,lp", [(40, 24, 8, 8, False), (36, 20, 10, 16, True), (24, 16, 8, 4, False),
                                         (70, 34, 8, 32, False), (72, 36, 10, 32, True)])
def test_block_checks_brute_force(oracle_mod, W, H, bd, w, lp):
    """The oracle's per-block test outputs (SURVEY 8(c) "Whole pipeline": AC checksum
    sum_{(i,j)!=(0,0)} C_ij (i n + j + 1), sample sum, H) against an independent computation:
    numpy.pad(edge) blocks, reshape-sum low-pass, exact object-integer T X T^T with the basis
    rebuilt from scipy's orthonormal DCT-II (rint(64 sqrt(n) Phi)), fsum H -- on 2 frames of
    ragged geometry (partial last block row and column)."""
    rng = np.random.default_rng(W * H + bd + w)
    hi = (1 << bd) - 1
    dt = np.uint8 if bd == 8 else np.uint16
    F = 2
    Y = rng.integers(0, hi + 1, size=(F, H, W)).astype(dt)
    U = rng.integers(0, hi + 1, size=(F, H // 2, W // 2)).astype(dt)
    V = rng.integers(0, hi + 1, size=(F, H // 2, W // 2)).astype(dt)
    _, checks = oracle_mod.analyze(Y, U, V, bd, w, lp, want_checks=True)
    wc = max(4, w // 2)
    for p, (plane, wp) in enumerate(((Y, w), (U, wc), (V, wc))):
        n = wp // 2 if lp else wp
        T = np.rint(64.0 * math.sqrt(n) * ortho_basis(n)).astype(np.int64).astype(object)
        rows, cols = -(-plane.shape[1] // wp), -(-plane.shape[2] // wp)
        for t in range(F):
            padded = np.pad(plane[t].astype(np.int64), ((0, rows * wp - plane.shape[1]), (0, cols * wp - plane.shape[2])),
                            mode="edge")
            k = 0
            for r in range(rows):
                for c in range(cols):
                    X = padded[r * wp:(r + 1) * wp, c * wp:(c + 1) * wp]
                    if lp:
                        X = (X.reshape(n, 2, n, 2).sum(axis=(1, 3)) + 2) // 4
                    Cm = T.dot(X.astype(object)).dot(T.T)
                    chk = sum(int(Cm[i, j]) * (i * n + j + 1) for i in range(n) for j in range(n) if (i, j) != (0, 0))
                    assert checks[p]["chk"][t, k] == chk, (p, t, r, c)
                    assert checks[p]["sumx"][t, k] == int(X.sum())
                    assert checks[p]["H"][t, k] == pytest.approx(brute_H(Cm.tolist(), n), rel=1e-13, abs=1e-300)
                    k += 1
            assert k == checks[p]["chk"].shape[1]
