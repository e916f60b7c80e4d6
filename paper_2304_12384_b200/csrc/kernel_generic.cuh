// kernel_generic.cuh -- the CUDA-core kernels for what the fused tensor-core kernel does
// not specialise: small_block_kernel (thread per 4 x 4 block, the w = 4 family, whose
// chroma grid differs from the luma grid: chroma block floor 4) and the reference
// warp-per-block kernel for every (block size, low-pass, bit depth) combination
// (VCA_FORCE_GENERIC builds; kept as a second, independent CUDA path for tests).  One warp computes one block of one plane of one frame:
//   A2 gather with edge replication, A3 low-pass (s+2)>>2 (R-5),
//   A4 C = T X T^T exact (int32 first pass, int64 second pass; R-1),
//   A5/A6 H and L in FP64 (R-2, R-3).
// Per-block (H, L) go to the partial-sum buffer (one entry per block), so the
// per-frame reduction order is fixed by the finalize kernel (R-11).
#pragma once
#include "vca_common.cuh"

namespace vca {

struct Planes3 {
    PlaneDesc p[3];
};

// Test-only outputs of the DUMP kernel instantiations (vca_debug_dump, vca_debug_analyze).
// Every array is indexed by the block's global index t * count[p] + k (frame t, raster block
// k); a NULL pointer is never written.  chk accumulates, with integer atomics (exact and
// order-independent), the checksum sum_{(i,j) != (0,0)} C_ij (i n + j + 1) mod 2^64 of each
// block's AC coefficients; the host zeroes it first.
struct DumpPtrs {
    int on;                     // launch the DUMP instantiation
    int32_t *coeffs[3];         // [F][C_p][n][n] (C_00 mod 2^32, R-11)
    int64_t *sumx[3];           // [F][C_p] sum of the DCT input samples (= C_00 / 4096)
    double *H[3];               // [F][C_p] texture energy
    double *L[3];               // [F][C_p] luminescence
    unsigned long long *chk[3];  // [F][C_p] AC checksum
};

__device__ __forceinline__ void chk_add(unsigned long long *chk, int64_t idx, int64_t v)
{
    if (chk && v) atomicAdd(chk + idx, (unsigned long long)v);
}

// Coefficient mutation for the suite's self-test (tests/test_mutation_gpu.py): a VCA_MUTATE
// build adds 1 to the coefficient at position pos of block `block` (global index) of plane
// `plane` in the instantiations selected by `which` (bit 0 production, bit 1 DUMP), as set by
// vca_debug_mutate.  Default builds compile mutate() to the identity.
#ifdef VCA_MUTATE
struct MutSpec {
    int plane, which, pos;
    long long block;
};
__device__ MutSpec vca_mut = {-1, 0, -1, -1};
constexpr bool kMutate = true;
template <bool DUMP>
__device__ __forceinline__ int32_t mutate(int32_t c, int plane, int64_t block, int pos)
{
    const MutSpec m = vca_mut;
    return (m.plane == plane && m.block == block && m.pos == pos && (m.which & (DUMP ? 2 : 1))) ? c + 1 : c;
}
#else
constexpr bool kMutate = false;
template <bool DUMP>
__device__ __forceinline__ int32_t mutate(int32_t c, int, int64_t, int)
{
    return c;
}
#endif

template <int BD>
__device__ __forceinline__ int load_sample(const uint8_t *frame, const PlaneDesc &P, int x, int y)
{
    x = min(max(x, 0), P.width - 1);   // edge replication
    y = min(max(y, 0), P.height - 1);
    const uint8_t *row = frame + (int64_t)y * P.pitch;
    if (BD == 8) return (int)__ldg(row + x);
    int v = (int)__ldg(reinterpret_cast<const uint16_t *>(row) + x);
    return min(v, 1023);                // 10-bit clamp
}

constexpr int kGenericWarps = 4;

template <int BD>
__global__ void __launch_bounds__(32 * kGenericWarps)
generic_block_kernel(Planes3 planes, int n_frames, int lowpass, const int8_t *__restrict__ T_all,
                     const double *__restrict__ W_all, Scratch s, DumpPtrs dump)
{
    __shared__ int32_t sX[kGenericWarps][32][33];
    __shared__ int32_t sZ[kGenericWarps][32][33];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int64_t C0 = planes.p[0].count, C1 = planes.p[1].count, C2 = planes.p[2].count;
    const int64_t Ctot = C0 + C1 + C2;
    const int64_t total = (int64_t)n_frames * Ctot;
    int32_t(*X)[33] = sX[wib];
    int32_t(*Z)[33] = sZ[wib];

    for (int64_t task = (int64_t)blockIdx.x * kGenericWarps + wib; task < total;
         task += (int64_t)gridDim.x * kGenericWarps) {
        const int64_t f = task / Ctot;
        int64_t k = task - f * Ctot;
        int p = 0;
        if (k >= C0) { k -= C0; p = 1; if (k >= C1) { k -= C1; p = 2; } }
        const PlaneDesc &P = planes.p[p];
        const int r = (int)(k / P.cols), c = (int)(k - (int64_t)r * P.cols);
        const uint8_t *frame = P.base + f * P.fstride;
        const int w = P.w, n = P.n;
        const int8_t *T = T_all + table_offset(n);
        const double *W = W_all + table_offset(n);

        // A2 + A3: gather the block (edge-replicated), low-pass if enabled
        for (int idx = lane; idx < n * n; idx += 32) {
            const int y = idx / n, x = idx - (idx / n) * n;
            int v;
            if (lowpass) {
                const int xs = c * w + 2 * x, ys = r * w + 2 * y;
                const int sum = load_sample<BD>(frame, P, xs, ys) + load_sample<BD>(frame, P, xs + 1, ys) +
                                load_sample<BD>(frame, P, xs, ys + 1) + load_sample<BD>(frame, P, xs + 1, ys + 1);
                v = (sum + 2) >> 2;
            } else {
                v = load_sample<BD>(frame, P, c * w + x, r * w + y);
            }
            X[y][x] = v;
        }
        __syncwarp();
        // A4 first pass: Z[i][x] = sum_y T[i][y] X[y][x]  (|Z| <= 32*1023*90 < 2^22: exact int32)
        for (int idx = lane; idx < n * n; idx += 32) {
            const int i = idx / n, x = idx - (idx / n) * n;
            int32_t acc = 0;
            for (int y = 0; y < n; ++y) acc += (int32_t)__ldg(T + i * n + y) * X[y][x];
            Z[i][x] = acc;
        }
        __syncwarp();
        // A4 second pass: C[i][j] = sum_x Z[i][x] T[j][x] (int64), then A5
        double hacc = 0.0;
        int64_t c00 = 0, ck = 0;
        const int64_t kg = f * P.count + k;  // global block index of the test outputs
        for (int idx = lane; idx < n * n; idx += 32) {
            const int i = idx / n, j = idx - (idx / n) * n;
            int64_t acc = 0;
            for (int x = 0; x < n; ++x) acc += (int64_t)Z[i][x] * (int64_t)__ldg(T + j * n + x);
            if (kMutate && idx != 0) acc = dump.on ? mutate<true>((int32_t)acc, p, kg, idx) : mutate<false>((int32_t)acc, p, kg, idx);
            if (idx == 0) c00 = acc;
            else ck += acc * (idx + 1);
            const int64_t a = acc < 0 ? -acc : acc;
            hacc += __ldg(W + idx) * (double)a;   // W(0,0) = 0 excludes DC
            if (dump.coeffs[p])
                dump.coeffs[p][kg * n * n + idx] = (int32_t)(uint32_t)(uint64_t)acc;
        }
        if (dump.on) chk_add(dump.chk[p], kg, ck);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hacc += __shfl_xor_sync(0xffffffffu, hacc, o);
        if (lane == 0) {
            const int64_t sumx = c00 >> 12;                 // C_00 = 4096 * sum(X) exactly
            const double L = sqrt((double)sumx / (double)n); // A6: sqrt(C_00 / (4096 n))
            double *pp = s.partial + (((int64_t)f * 3 + p) * s.P + k) * 2;
            pp[0] = hacc;
            pp[1] = L;
            if (p == 0) s.HY[f * C0 + k] = hacc;
            if (dump.sumx[p]) dump.sumx[p][kg] = sumx;
            if (dump.H[p]) dump.H[p][kg] = hacc;
            if (dump.L[p]) dump.L[p][kg] = L;
        }
        __syncwarp();
    }
}

// Thread-per-block kernel for the n = 4 family (w = 4 full; its chroma grid differs from
// the luma grid, so the fused kernel's units do not apply).  One warp takes a chunk of 32
// consecutive blocks of one plane of one frame (chunks never cross planes), one lane per
// 4 x 4 block, so a warp's row loads are 128 (8-bit) or 256 (10-bit) contiguous bytes; the
// (frame, plane, chunk) tasks are flattened so every warp stays busy across frames.
// A4 exact: the horizontal pass Z[y][j] = sum_x X[y][x] T[j][x] is a byte dot product of the
// packed row with the packed basis row (one IDP.4A, u8 x s8; 10-bit: two IDP.2A, u16 x s8),
// the vertical pass C[i][j] = sum_y T[i][y] Z[y][j] is int32 IMAD (|C| <= 256^2 * 1023 < 2^27);
// FP64 H and L.  The chunk's 32 (H, L) pairs are reduced in a fixed xor order and written as
// ONE partial (the finalize then adds ceil(C_p / 32) partials per plane in index order), so
// the per-block write traffic is only H_Y (needed for h).  DUMP: the test-only coefficient dump.
__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c)
{
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ int dp2a_us(uint32_t lo, uint32_t hi, uint32_t b)
{
    int d;
    asm("dp2a.lo.u32.s32 %0, %1, %2, 0;\n\tdp2a.hi.u32.s32 %0, %3, %2, %0;" : "=&r"(d) : "r"(lo), "r"(b), "r"(hi));
    return d;
}

#ifndef VCA_W4_B
#define VCA_W4_B 1  // 4 x 4 blocks per lane per chunk (chunk = 32 VCA_W4_B blocks; A/B: 2 and 4 -30 %)
#endif

#ifndef VCA_W4_MINB
#define VCA_W4_MINB 8  // 8 CTAs x 256 threads per SM: 32 registers (A/B: 1080p 192k -> 214k fps vs the default budget)
#endif
template <int BD, bool DUMP>
__global__ void __launch_bounds__(256, VCA_W4_MINB)
small_block_kernel(Planes3 planes, int n_frames, const int8_t *__restrict__ T_all, const double *__restrict__ W_all,
                   Scratch s, DumpPtrs dump)
{
    int T[4][4];
    uint32_t Tp[4];  // basis rows packed as s8 x 4
    double Wt[4][4];
    const int8_t *T4 = T_all + table_offset(4);
    const double *W4 = W_all + table_offset(4);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        Tp[i] = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            T[i][j] = (int)__ldg(T4 + i * 4 + j);
            Tp[i] |= (uint32_t)(T[i][j] & 255) << (8 * j);
            Wt[i][j] = __ldg(W4 + i * 4 + j);
        }
    }
    // 32-bit block indices within a frame (C_Y + C_U + C_V < 2^31, checked on the host)
    const int C0 = (int)planes.p[0].count, C1 = (int)planes.p[1].count, C2 = (int)planes.p[2].count;
    constexpr int CHB = 32 * VCA_W4_B;  // blocks per chunk
    const int CH0 = (C0 + CHB - 1) / CHB, CH1 = (C1 + CHB - 1) / CHB, CH2 = (C2 + CHB - 1) / CHB;
    const int CHtot = CH0 + CH1 + CH2;
    const int64_t tasks = (int64_t)n_frames * CHtot;
    const int lane = threadIdx.x & 31;
    const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t task = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); task < tasks;
         task += wstride) {
        const int f = (int)(task / CHtot);
        int ch = (int)(task - (int64_t)f * CHtot), p = 0;
        if (ch >= CH0) { ch -= CH0; p = 1; if (ch >= CH1) { ch -= CH1; p = 2; } }
        // plane fields by selects (a dynamically indexed parameter array would go to local memory)
        PlaneDesc P = planes.p[0];
        if (p == 1) P = planes.p[1];
        if (p == 2) P = planes.p[2];
        const int Cp = p == 0 ? C0 : p == 1 ? C1 : C2;
        double h = 0.0, L = 0.0;
#pragma unroll
        for (int b = 0; b < VCA_W4_B; ++b) {
            const int k = (ch * VCA_W4_B + b) * 32 + lane;
            if (k < Cp) {
                double hb = 0.0;
                const int r = k / P.cols, c = k - r * P.cols;
                const uint8_t *frame = P.base + (int64_t)f * P.fstride;
                // A2 gather (edge replication; 10-bit clamp) + A4 horizontal pass
                int Z[4][4];  // Z[y][j]
                const bool whole = c * 4 + 3 < P.width;
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    const int yy = min(r * 4 + y, P.height - 1);
                    const uint8_t *row = frame + (int64_t)yy * P.pitch;
                    if (BD == 8) {
                        uint32_t v;
                        if (whole) {
                            v = *reinterpret_cast<const uint32_t *>(row + 4 * c);
                        } else {
                            v = 0;
#pragma unroll
                            for (int x = 0; x < 4; ++x) v |= (uint32_t)load_sample<8>(frame, P, c * 4 + x, yy) << (8 * x);
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) Z[y][j] = dp4a_us(v, Tp[j], 0);
                    } else {
                        uint32_t lo, hi;
                        if (whole) {
                            const uint2 v = *reinterpret_cast<const uint2 *>(row + 8 * c);
                            lo = __vminu2(v.x, 0x03FF03FFu);
                            hi = __vminu2(v.y, 0x03FF03FFu);
                        } else {
                            lo = (uint32_t)load_sample<10>(frame, P, c * 4, yy) |
                                 ((uint32_t)load_sample<10>(frame, P, c * 4 + 1, yy) << 16);
                            hi = (uint32_t)load_sample<10>(frame, P, c * 4 + 2, yy) |
                                 ((uint32_t)load_sample<10>(frame, P, c * 4 + 3, yy) << 16);
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) Z[y][j] = dp2a_us(lo, hi, Tp[j]);
                    }
                }
                // A4 vertical pass, A5 (row-major, DC excluded)
                int c00 = 0;
                int64_t ck = 0;
                const int64_t kg = (int64_t)f * Cp + k;  // global block index of the test outputs
                int32_t *dco = nullptr;
                if (DUMP) dco = p == 0 ? dump.coeffs[0] : p == 1 ? dump.coeffs[1] : dump.coeffs[2];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        int cij = T[i][0] * Z[0][j] + T[i][1] * Z[1][j] + T[i][2] * Z[2][j] + T[i][3] * Z[3][j];
                        if (kMutate && (i | j)) cij = mutate<DUMP>(cij, p, kg, i * 4 + j);
                        if (i == 0 && j == 0) c00 = cij;
                        else hb = fma(Wt[i][j], (double)(cij < 0 ? -cij : cij), hb);
                        if (DUMP) {
                            if (i | j) ck += (int64_t)cij * (i * 4 + j + 1);
                            if (dco) dco[kg * 16 + i * 4 + j] = cij;
                        }
                    }
                const int64_t sumx = c00 >> 12;         // C_00 = 4096 * sum(X) exactly
                const double Lb = sqrt((double)sumx / 4.0);  // A6
                h += hb;  // per lane: block b = 0, 1, ... in order
                L += Lb;
                if (p == 0) s.HY[(int64_t)f * C0 + k] = hb;
                if (DUMP) {  // test outputs (NULL planes are skipped)
                    int64_t *sx = p == 0 ? dump.sumx[0] : p == 1 ? dump.sumx[1] : dump.sumx[2];
                    double *hh = p == 0 ? dump.H[0] : p == 1 ? dump.H[1] : dump.H[2];
                    double *ll = p == 0 ? dump.L[0] : p == 1 ? dump.L[1] : dump.L[2];
                    if (sx) sx[kg] = sumx;
                    if (hh) hh[kg] = hb;
                    if (ll) ll[kg] = Lb;
                    chk_add(p == 0 ? dump.chk[0] : p == 1 ? dump.chk[1] : dump.chk[2], kg, ck);
                }
            }
        }
        // A7 input: the chunk's fixed-order partial (xor tree over the 32 blocks)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            h += __shfl_xor_sync(0xffffffffu, h, o);
            L += __shfl_xor_sync(0xffffffffu, L, o);
        }
        if (lane == 0) {
            double *pp = s.partial + (((int64_t)f * 3 + p) * s.P + ch) * 2;
            pp[0] = h;
            pp[1] = L;
        }
    }
}

}  // namespace vca
