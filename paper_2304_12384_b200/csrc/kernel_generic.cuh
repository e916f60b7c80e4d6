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

struct DumpPtrs {
    int32_t *coeffs[3];
    int64_t *sumx[3];
    double *H[3];
    double *L[3];
};

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
        int64_t c00 = 0;
        for (int idx = lane; idx < n * n; idx += 32) {
            const int i = idx / n, j = idx - (idx / n) * n;
            int64_t acc = 0;
            for (int x = 0; x < n; ++x) acc += (int64_t)Z[i][x] * (int64_t)__ldg(T + j * n + x);
            if (idx == 0) c00 = acc;
            const int64_t a = acc < 0 ? -acc : acc;
            hacc += __ldg(W + idx) * (double)a;   // W(0,0) = 0 excludes DC
            if (dump.coeffs[p])
                dump.coeffs[p][k * n * n + idx] = (int32_t)(uint32_t)(uint64_t)acc;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hacc += __shfl_xor_sync(0xffffffffu, hacc, o);
        if (lane == 0) {
            const int64_t sumx = c00 >> 12;                 // C_00 = 4096 * sum(X) exactly
            const double L = sqrt((double)sumx / (double)n); // A6: sqrt(C_00 / (4096 n))
            double *pp = s.partial + (((int64_t)f * 3 + p) * s.P + k) * 2;
            pp[0] = hacc;
            pp[1] = L;
            if (p == 0) s.HY[f * C0 + k] = hacc;
            if (dump.sumx[p]) {
                dump.sumx[p][k] = sumx;
                dump.H[p][k] = hacc;
                dump.L[p][k] = L;
            }
        }
        __syncwarp();
    }
}

// Thread-per-block kernel for the n = 4 family (w = 4 full; its chroma grid differs from
// the luma grid, so the fused kernel's units do not apply).  One thread computes one 4 x 4
// block of one plane of one frame; consecutive threads take consecutive blocks of a block
// row, so a warp's row loads are 128 (8-bit) or 256 (10-bit) contiguous bytes.  Same
// arithmetic as generic_block_kernel: exact int32 C = T X T^T (|C| <= 256^2 * 1023 < 2^27),
// FP64 H and L, one (H, L) partial per block for the fixed-order finalize.
template <int BD>
__global__ void __launch_bounds__(256)
small_block_kernel(Planes3 planes, int n_frames, const int8_t *__restrict__ T_all, const double *__restrict__ W_all,
                   Scratch s, DumpPtrs dump)
{
    int T[4][4];
    double Wt[4][4];
    const int8_t *T4 = T_all + table_offset(4);
    const double *W4 = W_all + table_offset(4);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            T[i][j] = (int)__ldg(T4 + i * 4 + j);
            Wt[i][j] = __ldg(W4 + i * 4 + j);
        }
    // 32-bit block indices within a frame (C_Y + C_U + C_V < 2^31, checked on the host),
    // frames in an outer loop: no 64-bit divisions on the per-block path
    const int C0 = (int)planes.p[0].count, C1 = (int)planes.p[1].count, C2 = (int)planes.p[2].count;
    const int Ctot = C0 + C1 + C2;
    const int stride = gridDim.x * blockDim.x;
    for (int f = 0; f < n_frames; ++f)
    for (int kk = blockIdx.x * blockDim.x + threadIdx.x; kk < Ctot; kk += stride) {
        int k = kk, p = 0;
        if (k >= C0) { k -= C0; p = 1; if (k >= C1) { k -= C1; p = 2; } }
        // plane fields by selects (a dynamically indexed parameter array would go to local memory)
        PlaneDesc P = planes.p[0];
        if (p == 1) P = planes.p[1];
        if (p == 2) P = planes.p[2];
        const int r = k / P.cols, c = k - r * P.cols;
        const uint8_t *frame = P.base + (int64_t)f * P.fstride;
        // A2: gather (edge replication; 10-bit clamp)
        int X[4][4];
        const bool whole = c * 4 + 3 < P.width;
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int yy = min(r * 4 + y, P.height - 1);
            const uint8_t *row = frame + (int64_t)yy * P.pitch;
            if (whole && BD == 8) {
                const uint32_t v = *reinterpret_cast<const uint32_t *>(row + 4 * c);
#pragma unroll
                for (int x = 0; x < 4; ++x) X[y][x] = (int)((v >> (8 * x)) & 255u);
            } else if (whole) {
                const uint2 v = *reinterpret_cast<const uint2 *>(row + 8 * c);
                X[y][0] = min((int)(v.x & 0xFFFFu), 1023);
                X[y][1] = min((int)(v.x >> 16), 1023);
                X[y][2] = min((int)(v.y & 0xFFFFu), 1023);
                X[y][3] = min((int)(v.y >> 16), 1023);
            } else {
#pragma unroll
                for (int x = 0; x < 4; ++x) X[y][x] = load_sample<BD>(frame, P, c * 4 + x, yy);
            }
        }
        // A4: Z[i][x] = sum_y T[i][y] X[y][x]; C[i][j] = sum_x Z[i][x] T[j][x]  (exact int32)
        int Z[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int x = 0; x < 4; ++x)
                Z[i][x] = T[i][0] * X[0][x] + T[i][1] * X[1][x] + T[i][2] * X[2][x] + T[i][3] * X[3][x];
        double h = 0.0;
        int c00 = 0;
        int32_t *const dco = p == 0 ? dump.coeffs[0] : p == 1 ? dump.coeffs[1] : dump.coeffs[2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cij = Z[i][0] * T[j][0] + Z[i][1] * T[j][1] + Z[i][2] * T[j][2] + Z[i][3] * T[j][3];
                if (i == 0 && j == 0) c00 = cij;
                else h = fma(Wt[i][j], (double)(cij < 0 ? -cij : cij), h);  // A5, row-major, DC excluded
                if (dco) dco[(int64_t)k * 16 + i * 4 + j] = cij;
            }
        const int64_t sumx = c00 >> 12;               // C_00 = 4096 * sum(X) exactly
        const double L = sqrt((double)sumx / 4.0);    // A6
        double *pp = s.partial + (((int64_t)f * 3 + p) * s.P + k) * 2;
        pp[0] = h;
        pp[1] = L;
        if (p == 0) s.HY[(int64_t)f * C0 + k] = h;
        if (dco) {  // debug dump (all three planes are dumped together)
            (p == 0 ? dump.sumx[0] : p == 1 ? dump.sumx[1] : dump.sumx[2])[k] = sumx;
            (p == 0 ? dump.H[0] : p == 1 ? dump.H[1] : dump.H[2])[k] = h;
            (p == 0 ? dump.L[0] : p == 1 ? dump.L[1] : dump.L[2])[k] = L;
        }
    }
}

}  // namespace vca
