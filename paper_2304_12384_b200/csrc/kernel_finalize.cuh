// kernel_finalize.cuh -- per-frame reduction and record emit (A7-A9).
// One CTA per frame: fixed-order reductions of the partial sums into
// E_p = sum H / (C_p n_p^2), L_p = sum L / C_p (R-6) and of the
// luma SAD into h = sum_k |H_t[k] - H_{t-1}[k]| / (C_Y n_Y^2) (R-7);
// record {poc, E_Y, h, L_Y, E_U, L_U, E_V, L_V}.
// The reduction order depends only on the frame's own data layout and the
// fixed block size (256), never on the grid, so records are bit-identical for
// any frame-range split.
#pragma once
#include "vca_common.cuh"
#include "../../include/vca.h"

namespace vca {

constexpr int kFinalizeThreads = 256;

struct FinalizeArgs {
    Scratch s;
    int n_frames, n_halo;
    int64_t count[3];
    int n[3];
    const double *prevHY;  // H_Y of the frame before frame 0 (carried), or nullptr
    double *saveHY;        // receives the last frame's H_Y (the next call's prevHY; another buffer)
    int64_t first_poc;
    vca_features *out;
    int frames_per_cta;    // consecutive frames per CTA (> 1 only when C_Y <= kFinalizeThreads * kHYRegs)
};

// A CTA that finalizes several consecutive frames keeps the previous frame's H_Y in registers
// (kHYRegs per thread), so each frame's H_Y is read from memory once instead of twice.
constexpr int kHYRegs = 32;

template <int K>
__device__ __forceinline__ void block_reduce(double (&v)[K], double (*sm)[kFinalizeThreads / 32])
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < K; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
        if (lane == 0) sm[q][wid] = v[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < K; ++q) {
        double x = lane < kFinalizeThreads / 32 ? sm[q][lane] : 0.0;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        v[q] = x;  // the total, in lanes 0..7 of every warp
    }
}

// One frame's record from its partial sums and h SAD (v[0..6]), fixed-order block reduction.
__device__ __forceinline__ void emit_record(const FinalizeArgs &a, int f, bool have_prev, double (&v)[7],
                                            double (*sm)[kFinalizeThreads / 32])
{
    block_reduce<7>(v, sm);
    if (threadIdx.x == 0 && f >= a.n_halo) {
        vca_features r;
        r.poc = a.first_poc + (f - a.n_halo);
        const double nY = (double)a.n[0], nU = (double)a.n[1], nV = (double)a.n[2];
        r.E_Y = v[0] / ((double)a.count[0] * nY * nY);
        r.L_Y = v[1] / (double)a.count[0];
        r.E_U = v[2] / ((double)a.count[1] * nU * nU);
        r.L_U = v[3] / (double)a.count[1];
        r.E_V = v[4] / ((double)a.count[2] * nV * nV);
        r.L_V = v[5] / (double)a.count[2];
        r.h = have_prev ? v[6] / ((double)a.count[0] * nY * nY) : 0.0;
        a.out[f - a.n_halo] = r;
    }
    __syncthreads();  // sm is reused by the next frame
}

__device__ __forceinline__ void partial_sums(const FinalizeArgs &a, int f, double (&v)[7])
{
#pragma unroll
    for (int q = 0; q < 7; ++q) v[q] = 0.0;
    // partial sums of the block kernel, plane by plane, in index order per thread
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        const double *pp = a.s.partial + ((int64_t)f * 3 + p) * a.s.P * 2;
        for (int q = threadIdx.x; q < a.s.Pp[p]; q += kFinalizeThreads) {
            v[2 * p] += pp[2 * q];
            v[2 * p + 1] += pp[2 * q + 1];
        }
    }
}

// MULTI = false: one frame per CTA (the default).  MULTI = true: a.frames_per_cta consecutive
// frames per CTA (A/B only, VCA_FIN_FRAMES > 1).  Separate instantiations: the register-resident
// H_Y of the multi-frame path (185 registers) would otherwise cap the one-frame kernel at one
// CTA per SM (measured: 16.4 -> 30.9 us per 600 frames).
template <bool MULTI>
__global__ void __launch_bounds__(kFinalizeThreads) finalize_kernel(FinalizeArgs a)
{
    __shared__ double sm[7][kFinalizeThreads / 32];
    const int tid = threadIdx.x;
    double v[7];
    {  // carry the last frame's H_Y to the next call (R-7): every CTA copies a slice
        const double *last = a.s.HY + (int64_t)(a.n_frames - 1) * a.count[0];
        const int64_t per = (a.count[0] + gridDim.x - 1) / gridDim.x;
        const int64_t k0 = (int64_t)blockIdx.x * per, k1 = min(a.count[0], k0 + per);
        for (int64_t k = k0 + tid; k < k1; k += kFinalizeThreads) a.saveHY[k] = last[k];
    }
    if (!MULTI) {
        const int f = blockIdx.x;
        partial_sums(a, f, v);
        // h: SAD against the previous frame's luma energies (R-7)
        const double *cur = a.s.HY + (int64_t)f * a.count[0];
        const double *prev = f > 0 ? cur - a.count[0] : a.prevHY;
        if (prev) {
            for (int64_t k = tid; k < a.count[0]; k += kFinalizeThreads) v[6] += fabs(cur[k] - prev[k]);
        }
        emit_record(a, f, prev != nullptr, v, sm);
    } else {
        // frames f0 .. f0 + frames_per_cta - 1: the previous frame's H_Y stays in registers (the same
        // per-thread index order k = tid + 256 i as above, so the sums are bit-identical)
        const int f0 = blockIdx.x * a.frames_per_cta;
        const int f1 = min(a.n_frames, f0 + a.frames_per_cta);
        const int C = (int)a.count[0];
        double hp[kHYRegs];
        const double *prev0 = f0 > 0 ? a.s.HY + (int64_t)(f0 - 1) * C : a.prevHY;
        bool have_prev = prev0 != nullptr;
#pragma unroll
        for (int i = 0; i < kHYRegs; ++i) {
            const int k = tid + i * kFinalizeThreads;
            hp[i] = (have_prev && k < C) ? prev0[k] : 0.0;
        }
        for (int f = f0; f < f1; ++f) {
            partial_sums(a, f, v);
            const double *cur = a.s.HY + (int64_t)f * C;
#pragma unroll
            for (int i = 0; i < kHYRegs; ++i) {
                const int k = tid + i * kFinalizeThreads;
                if (k < C) {
                    const double x = cur[k];
                    if (have_prev) v[6] += fabs(x - hp[i]);
                    hp[i] = x;
                }
            }
            emit_record(a, f, have_prev, v, sm);
            have_prev = true;
        }
    }
}

}  // namespace vca
