/*
 * vca_oracle.c -- plain, slow, obviously-correct CPU oracle for the VCA v2.0
 * hot path (arxiv 2304.12384).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * product path (paper_2304_12384_b200/csrc); neither includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * "R-k" = reading k listed in DESIGN.md section "Readings".
 *
 * What it computes (section 2: "seven blockwise
 * DCT-energy-based features E_Y, h, L_Y, E_U, E_V, L_U, L_V"; formulas
 * from SPEC.md features module S:191-235, integer transform per the
 * BASELINE.json north star):
 *
 *   for every frame, for every plane p in {Y,U,V}:
 *     1. block grid, edge replication
 *     2. optional 2x2 low-pass downsample        (R-5)
 *     3. integer 2-D DCT  C = T_n X T_n^T, int64 (R-1)
 *     4. H = sum_{(i,j)!=(0,0)} w_n(i,j) |C_ij/(4096 n)|  (R-2)
 *        L_blk = sqrt(C_00/(4096 n))             (R-2)
 *     5. E_p = sum_k H_k / (C_p n^2), L_p = sum_k L_k / C_p
 *     6. h   = sum_k |H_Y,t[k]-H_Y,t-1[k]| / (C_Y n^2), 0 at sequence start
 *
 *
 * Arithmetic: int64 for every integer, IEEE double for every real, every
 * sum sequential in raster / row-major order.  No blocking, no
 * fusion, no butterflies: the direct matrix product of the definition.
 * The only parallelism is OpenMP over frames for steps 1-5 (each frame is
 * computed by exactly the same sequential code); step 6 runs sequentially.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * (brute force, closed forms, SPEC.md worked examples) -- see DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define VO_OK 0
#define VO_EINVAL -1
#define VO_EBLOCK -2
#define VO_EBD -3
#define VO_ENOMEM -8

/* Per-frame record, CSV column order of S:456: POC,E_Y,h,L_Y,E_U,L_U,E_V,L_V */
typedef struct {
    int64_t poc;
    double E_Y, h, L_Y, E_U, L_U, E_V, L_V;
} vo_record;

/* R-1: T_n[k][x] = round(64 * sqrt(2) * c_k * cos(pi (2x+1) k / (2n))),
 * c_0 = 1/sqrt(2), c_k = 1 otherwise.  No entry lies near a rounding tie
 * (min distance 0.0082 at n=32), so lround is unambiguous. */
int vo_basis(int n, int32_t *T)
{
    if (!(n == 4 || n == 8 || n == 16 || n == 32) || !T) return VO_EBLOCK;
    const double pi = 3.14159265358979323846;
    for (int k = 0; k < n; ++k) {
        double ck = (k == 0) ? (1.0 / sqrt(2.0)) : 1.0;
        for (int x = 0; x < n; ++x) {
            double v = 64.0 * sqrt(2.0) * ck * cos(pi * (2.0 * x + 1.0) * k / (2.0 * n));
            T[k * n + x] = (int32_t)lround(v);
        }
    }
    return VO_OK;
}

/* weight(i,j) = exp(|(i*j/n^2)^2 - 1|), n = DCT size (R-3). */
double vo_weight(int n, int i, int j)
{
    double r = ((double)i * (double)j) / ((double)n * (double)n);
    return exp(fabs(r * r - 1.0));
}

/* One sample of a plane with edge replication and the 10-bit
 * clamp.  8-bit planes are bytes, 10-bit planes are little-endian
 * uint16 containers. */
static int64_t vo_sample(const uint8_t *plane, int64_t pitch, int bd, int pw, int ph, int x, int y)
{
    if (x < 0) x = 0;
    if (x > pw - 1) x = pw - 1;
    if (y < 0) y = 0;
    if (y > ph - 1) y = ph - 1;
    const uint8_t *row = plane + (int64_t)y * pitch;
    if (bd == 8) return (int64_t)row[x];
    int64_t v = (int64_t)row[2 * x] | ((int64_t)row[2 * x + 1] << 8);
    if (v > 1023) v = 1023;
    return v;
}

/* Steps 1-4 for block (r, c) of one plane.  w = block size in samples.
 * Outputs: n (DCT size), coeffs[n*n] (optional, int64, row-major C[i][j],
 * i = vertical frequency, j = horizontal; R-4), *sumx = sum of the samples
 * entering the DCT (= C_00 / 4096), *H, *L. */
int vo_block(const uint8_t *plane, int64_t pitch, int bd, int pw, int ph, int w, int lowpass,
             int r, int c, int64_t *coeffs, int64_t *sumx, double *H, double *L)
{
    if (!(w == 4 || w == 8 || w == 16 || w == 32)) return VO_EBLOCK;
    if (lowpass && w < 8) return VO_EBLOCK;
    if (bd != 8 && bd != 10) return VO_EBD;
    int n = lowpass ? w / 2 : w;
    int64_t X[32][32];
    int64_t S[32][32];
    int32_t T[32 * 32];
    int64_t Z[32][32];
    int64_t C[32][32];

    /* step 1: gather the w x w block with edge replication */
    for (int y = 0; y < w; ++y)
        for (int x = 0; x < w; ++x)
            S[y][x] = vo_sample(plane, pitch, bd, pw, ph, c * w + x, r * w + y);

    /* step 2: low-pass -- pad then downsample, d = (s + 2) >> 2 with s the
     * 2x2 sum: the mean rounded half away from zero (R-5) */
    if (lowpass) {
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) {
                int64_t s = S[2 * y][2 * x] + S[2 * y][2 * x + 1] + S[2 * y + 1][2 * x] + S[2 * y + 1][2 * x + 1];
                X[y][x] = (s + 2) / 4; /* s >= 0: floor division == >> 2 */
            }
    } else {
        for (int y = 0; y < n; ++y)
            for (int x = 0; x < n; ++x) X[y][x] = S[y][x];
    }

    /* step 3: C = T X T^T, exact in int64, no intermediate shift (R-1) */
    vo_basis(n, T);
    for (int i = 0; i < n; ++i)
        for (int x = 0; x < n; ++x) {
            int64_t acc = 0;
            for (int y = 0; y < n; ++y) acc += (int64_t)T[i * n + y] * X[y][x];
            Z[i][x] = acc; /* Z = T X */
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            int64_t acc = 0;
            for (int x = 0; x < n; ++x) acc += Z[i][x] * (int64_t)T[j * n + x];
            C[i][j] = acc; /* C = Z T^T */
        }

    int64_t s = 0;
    for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) s += X[y][x];

    /* step 4: texture energy and luminescence in orthonormal units:
     * coefficient / (4096 n) (R-2); DC excluded from H. */
    double scale = 1.0 / (4096.0 * (double)n);
    double acc = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            if (i == 0 && j == 0) continue;
            int64_t a = C[i][j] < 0 ? -C[i][j] : C[i][j];
            acc += vo_weight(n, i, j) * ((double)a * scale);
        }
    if (coeffs)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) coeffs[i * n + j] = C[i][j];
    if (sumx) *sumx = s;
    if (H) *H = acc;
    if (L) *L = sqrt((double)C[0][0] * scale); /* sqrt(DC) */
    return VO_OK;
}

/* auto block size; chroma block = w/2, floor 4. */
int vo_resolve_block(int height, int block_size)
{
    if (block_size == 0) return height >= 2160 ? 32 : (height >= 1080 ? 16 : 8);
    return block_size;
}

int vo_chroma_block(int w)
{
    return w / 2 < 4 ? 4 : w / 2;
}

/* Block count C = ceil(pw/w) * ceil(ph/w). */
int64_t vo_block_count(int pw, int ph, int w)
{
    return (int64_t)((pw + w - 1) / w) * (int64_t)((ph + w - 1) / w);
}

/* Exact integer checks of one block's coefficients (test outputs, SURVEY 8(c)
 * "Whole pipeline"): the AC checksum sum_{(i,j) != (0,0)} C_ij * (i n + j + 1),
 * row-major; |C_ij| < 2^31 and n^2 <= 1024 terms, so the int64 sum is exact. */
static int64_t vo_checksum(const int64_t *coeffs, int n)
{
    int64_t acc = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (i != 0 || j != 0) acc += coeffs[i * n + j] * (int64_t)(i * n + j + 1);
    return acc;
}

/* Steps 1-5 for one plane of one frame: E_p, L_p and (optionally) the
 * per-block H vector in raster order, plus the optional per-block test
 * outputs chk (vo_checksum), sx (sum of the DCT input samples) and Hb (H). */
static int vo_plane(const uint8_t *plane, int64_t pitch, int bd, int pw, int ph, int w, int lowpass,
                    double *E, double *Lp, double *Hvec, int64_t *chk, int64_t *sx, double *Hb)
{
    int n = lowpass ? w / 2 : w;
    int cols = (pw + w - 1) / w, rows = (ph + w - 1) / w;
    int64_t C = (int64_t)cols * rows;
    double sumH = 0.0, sumL = 0.0;
    int64_t k = 0;
    int64_t coeffs[32 * 32];
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c, ++k) {
            double H, L;
            int64_t s = 0;
            int rc = vo_block(plane, pitch, bd, pw, ph, w, lowpass, r, c, chk ? coeffs : NULL, &s, &H, &L);
            if (rc) return rc;
            if (Hvec) Hvec[k] = H;
            if (chk) chk[k] = vo_checksum(coeffs, n);
            if (sx) sx[k] = s;
            if (Hb) Hb[k] = H;
            sumH += H;
            sumL += L;
        }
    *E = sumH / ((double)C * (double)n * (double)n);
    *Lp = sumL / (double)C;                          /* R-6 */
    return VO_OK;
}

/* Whole-sequence analysis (S:359 analyze_stream, S:227 analyze_frame).
 *
 * planes[p] points at frame 0 of plane p; frame t of plane p starts at
 * planes[p] + t * frame_stride[p]; rows are pitch[p] bytes apart.
 * n_halo (0 or 1): frame 0 only provides H_Y,t-1 for frame 1 and emits no
 * record.  prev_HY (length C_Y, may be NULL): H_Y of the frame before
 * frame 0; NULL with n_halo == 0 means frame 0 starts a sequence (h = 0).
 * Records are written for frames n_halo..n_frames-1 with poc = first_poc + i.
 * out_HY (optional) receives H_Y for all n_frames frames, [n_frames][C_Y].
 * n_threads <= 0 means the OpenMP default. */
int vo_analyze_checks(const uint8_t *const planes[3], const int64_t pitch[3], const int64_t frame_stride[3],
                      int width, int height, int bd, int block_size, int lowpass, int n_frames, int n_halo,
                      const double *prev_HY, int64_t first_poc, vo_record *out, double *out_HY, int n_threads,
                      int64_t *const chk[3], int64_t *const sx[3], double *const Hb[3]);

int vo_analyze(const uint8_t *const planes[3], const int64_t pitch[3], const int64_t frame_stride[3],
               int width, int height, int bd, int block_size, int lowpass, int n_frames, int n_halo,
               const double *prev_HY, int64_t first_poc, vo_record *out, double *out_HY, int n_threads)
{
    return vo_analyze_checks(planes, pitch, frame_stride, width, height, bd, block_size, lowpass, n_frames,
                             n_halo, prev_HY, first_poc, out, out_HY, n_threads, NULL, NULL, NULL);
}

/* vo_analyze plus optional per-block test outputs for every frame t and plane
 * p with non-NULL chk/sx/Hb (arrays of n_frames * C_p entries, index
 * t * C_p + k): the AC checksum, the sample sum and H of every block. */
int vo_analyze_checks(const uint8_t *const planes[3], const int64_t pitch[3], const int64_t frame_stride[3],
                      int width, int height, int bd, int block_size, int lowpass, int n_frames, int n_halo,
                      const double *prev_HY, int64_t first_poc, vo_record *out, double *out_HY, int n_threads,
                      int64_t *const chk[3], int64_t *const sx[3], double *const Hb[3])
{
    if (!planes || !pitch || !frame_stride || !out) return VO_EINVAL;
    if (width < 2 || height < 2 || (width & 1) || (height & 1)) return VO_EINVAL;
    if (bd != 8 && bd != 10) return VO_EBD;
    if (n_halo < 0 || n_halo > 1 || n_frames < 1 + n_halo) return VO_EINVAL;
    int w = vo_resolve_block(height, block_size);
    if (!(w == 4 || w == 8 || w == 16 || w == 32)) return VO_EBLOCK;
    int wc = vo_chroma_block(w);
    if (lowpass && (w < 8 || wc < 8)) return VO_EBLOCK;
    int nY = lowpass ? w / 2 : w, nC = lowpass ? wc / 2 : wc;
    (void)nC;
    int pw[3] = {width, width / 2, width / 2}, ph[3] = {height, height / 2, height / 2};
    int wp[3] = {w, wc, wc};
    int64_t CY = vo_block_count(width, height, w);

    double *HY = (double *)malloc(sizeof(double) * (size_t)CY * (size_t)n_frames);
    double *feat = (double *)malloc(sizeof(double) * 6 * (size_t)n_frames);
    if (!HY || !feat) {
        free(HY);
        free(feat);
        return VO_ENOMEM;
    }
    int err = VO_OK;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int t = 0; t < n_frames; ++t) {
        for (int p = 0; p < 3; ++p) {
            const uint8_t *base = planes[p] + (int64_t)t * frame_stride[p];
            double E = 0.0, L = 0.0;
            const int64_t Cp = vo_block_count(pw[p], ph[p], wp[p]);
            const size_t o = (size_t)t * (size_t)Cp;
            int rc = vo_plane(base, pitch[p], bd, pw[p], ph[p], wp[p], lowpass, &E, &L,
                              p == 0 ? HY + (size_t)t * (size_t)CY : NULL, chk && chk[p] ? chk[p] + o : NULL,
                              sx && sx[p] ? sx[p] + o : NULL, Hb && Hb[p] ? Hb[p] + o : NULL);
            if (rc) err = rc;
            feat[6 * t + 2 * p] = E;
            feat[6 * t + 2 * p + 1] = L;
        }
    }
    if (err) {
        free(HY);
        free(feat);
        return err;
    }
    /* step 6, sequential over frames */
    for (int t = n_halo; t < n_frames; ++t) {
        const double *cur = HY + (size_t)t * (size_t)CY;
        const double *prev = t > 0 ? HY + (size_t)(t - 1) * (size_t)CY : prev_HY;
        double h = 0.0;
        if (prev) {
            double s = 0.0;
            for (int64_t k = 0; k < CY; ++k) s += fabs(cur[k] - prev[k]);
            h = s / ((double)CY * (double)nY * (double)nY);
        }
        vo_record *o = out + (t - n_halo);
        o->poc = first_poc + (t - n_halo);
        o->E_Y = feat[6 * t + 0];
        o->L_Y = feat[6 * t + 1];
        o->E_U = feat[6 * t + 2];
        o->L_U = feat[6 * t + 3];
        o->E_V = feat[6 * t + 4];
        o->L_V = feat[6 * t + 5];
        o->h = h;
    }
    if (out_HY) memcpy(out_HY, HY, sizeof(double) * (size_t)CY * (size_t)n_frames);
    free(HY);
    free(feat);
    return VO_OK;
}
