// Measured prototype of the tcgen05 path for the n = 32 DCT (NEXT-1, config 2's luma): the compute
// pipeline of an exact 32x32 integer DCT + FP64 texture energy on the 5th-gen tensor cores,
// isolated from memory (pixels stay in shared memory), to compare with the mma.sync kernel.
//
// Tile = 4 luma blocks of one block row (M = 128 TMEM lanes = (block b, frequency k)):
//   pass 1 (TS):  D1[(b,k)][y] = sum_(b',x) A1[(b,k)][(b',x)] . X_b'[y][x]
//                 A1 = blockdiag(T,T,T,T) resident in TMEM (4 K-steps of 32 bytes), B = the pixel
//                 rows (K-major, the 4 blocks' row y side by side) in shared memory;
//   split:        each epilogue thread (lane (b,k)) loads its 32 values of y, splits them into three
//                 byte planes packed 4 y per word and writes them back to its own TMEM lane
//                 (tcgen05.st) -- no transpose: the lane is already (b,k);
//   pass 2 (TS):  D2p[(b,k)][i] = sum_y plane_p[(b,k)][y] . T[i][y]   (p = 0, 1, 2; B = T in smem)
//   epilogue:     C = D20 + 2^8 D21 + 2^16 D22 (= C_b[i][k]), H_b += w(i,k) |C| / (4096 n) in FP64.
// One thread issues the MMAs; NSETS sets of 4 epilogue warps each own a TMEM slot and take tiles
// round robin.  Checks the H of one tile against a host computation (exact integer DCT + FP64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_dct32 tc_dct32.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                         \
        }                                                                                    \
    } while (0)

#ifndef NSETS
#define NSETS 3
#endif
constexpr int kSlot = 160;  // TMEM columns per slot: D1 32 | A2 24 (+8 pad) | D2 96

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_s8, bool b_s8)
{
    return (2u << 4) | ((a_s8 ? 1u : 0u) << 7) | ((b_s8 ? 1u : 0u) << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P;\nW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra W_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#define LD32(addr, r)                                                                                              \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"  \
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                       \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),      \
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),      \
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                            \
                 : "r"(addr))
#define ST8(addr, w)                                                                                            \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(w[0]), \
                 "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])                   \
                 : "memory")

// K-major canonical no-swizzle offset (8-bit): core (r/8, k/16) at (r/8) SBO + (k/16) LBO
__host__ __device__ inline int kmaj(int r, int k, int lbo, int sbo) { return (r / 8) * sbo + (k / 16) * lbo + (r % 8) * 16 + (k % 16); }

struct Smem {
    uint8_t B1[32 * 128];  // pixels: rows y (N = 32), K = (b', x) 128 bytes; LBO 128, SBO 1024
    uint8_t B2[32 * 32];   // T: rows i (N = 32), K = y 32 bytes; LBO 128, SBO 256
    double Wt[32 * 32];    // w(i,k) / (4096 n) at [i][k]
    uint64_t d1[NSETS], a2[NSETS], d2[NSETS], fr[NSETS];
    uint32_t tbase;
};

__global__ void __launch_bounds__(32 * (1 + 4 * NSETS), 1)
k_dct32(const int8_t *T, const uint8_t *X, const double *W, int tiles, double *Hout, long long *cycles)
{
    extern __shared__ __align__(1024) uint8_t dyn[];
    Smem &S = *reinterpret_cast<Smem *>(dyn);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 32 * 128; i += blockDim.x) {
        const int y = i / 128, k = i % 128;  // k = (b', x)
        S.B1[kmaj(y, k, 128, 1024)] = X[(k / 32) * 1024 + y * 32 + (k % 32)];
    }
    for (int i = tid; i < 32 * 32; i += blockDim.x) {
        const int r = i / 32, k = i % 32;
        S.B2[kmaj(r, k, 128, 256)] = (uint8_t)T[r * 32 + k];
        S.Wt[i] = W[i];
    }
    if (tid == 0) {
        for (int s = 0; s < NSETS; ++s) {
            mbar_init(&S.d1[s], 1);
            mbar_init(&S.a2[s], 128);
            mbar_init(&S.d2[s], 1);
            mbar_init(&S.fr[s], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&S.tbase))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = S.tbase;
    // A1 = blockdiag(T x 4) into TMEM columns [0, 32): the first epilogue set writes it
    if (warp >= 1 && warp <= 4) {
        const int b = warp & 3, k = lane;  // a warp reaches TMEM lanes 32 (warp % 4) .. + 31: lane 32 b + k
        const uint32_t lanebase = tm + ((uint32_t)(32 * b) << 16);
        for (int cb = 0; cb < 4; ++cb) {
            uint32_t w[8];
            for (int c = 0; c < 8; ++c) {
                uint32_t v = 0;
                for (int q = 0; q < 4; ++q) {
                    const int kk = cb * 32 + 4 * c + q;  // K index (b', x)
                    const int bp = kk / 32, x = kk % 32;
                    const int t = bp == b ? (int)T[k * 32 + x] : 0;
                    v |= (uint32_t)(t & 255) << (8 * q);
                }
                w[c] = v;
            }
            ST8(lanebase + 8 * cb, w);
        }
        wait_st();
    }
    fence_before();
    __syncthreads();
    fence_after();
    long long t0 = clock64();
    if (warp == 0) {
        // ---- MMA issuer: pass 1 of tile t, then pass 2 of tile t - 1
        if (lane == 0) {
            const uint32_t id1 = idesc_i8(128, 32, true, false);   // A = T (s8), B = pixels (u8)
            const uint64_t b1 = sdesc(smem_u32(S.B1), 128, 1024);
            const uint64_t b2 = sdesc(smem_u32(S.B2), 128, 256);
            for (int t = 0; t <= tiles; ++t) {
                if (t < tiles) {
                    const int s = t % NSETS, use = t / NSETS;
                    if (use > 0) mbar_wait(&S.fr[s], (use - 1) & 1);
                    fence_after();
                    const uint32_t D1 = tm + 32 + s * kSlot;
#pragma unroll
                    for (int kb = 0; kb < 4; ++kb)  // K-steps over b': A1 columns 8 kb, B bytes 32 kb
                        mma_ts(D1, tm + 8 * kb, b1 + (uint64_t)(kb * 16), id1, kb);  // +256 B = 2 K chunks
                    commit(&S.d1[s]);
                }
                if (t >= 1) {
                    const int tp = t - 1, s = tp % NSETS, use = tp / NSETS;
                    mbar_wait(&S.a2[s], use & 1);
                    fence_after();
                    const uint32_t A2 = tm + 32 + s * kSlot + 32, D2 = tm + 32 + s * kSlot + 64;
#pragma unroll
                    for (int p = 0; p < 3; ++p)
                        mma_ts(D2 + 32 * p, A2 + 8 * p, b2, idesc_i8(128, 32, p == 2, true), 0);
                    commit(&S.d2[s]);
                }
            }
        }
    } else {
        // ---- epilogue sets: set e = (warp - 1) / 4 takes tiles e, e + NSETS, ...
        const int e = (warp - 1) >> 2, b = warp & 3, k = lane;  // TMEM lane quadrant = warp % 4
        const uint32_t lane_off = (uint32_t)(32 * b) << 16;
        double H = 0.0;
        for (int t = e; t < tiles; t += NSETS) {
            const int use = t / NSETS;
            const uint32_t base = tm + lane_off + 32 + e * kSlot;
            mbar_wait(&S.d1[e], use & 1);
            fence_after();
            uint32_t z[32];
            LD32(base, z);
            wait_ld();
            uint32_t w0[8], w1[8], w2[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t v0 = z[4 * c], v1 = z[4 * c + 1], v2 = z[4 * c + 2], v3 = z[4 * c + 3];
                const uint32_t s0 = __byte_perm(v0, v1, 0x5140), s1 = __byte_perm(v0, v1, 0x7362);
                const uint32_t s2 = __byte_perm(v2, v3, 0x5140), s3 = __byte_perm(v2, v3, 0x7362);
                w0[c] = __byte_perm(s0, s2, 0x5410);
                w1[c] = __byte_perm(s0, s2, 0x7632);
                w2[c] = __byte_perm(s1, s3, 0x5410);
            }
            ST8(base + 32, w0);
            ST8(base + 40, w1);
            ST8(base + 48, w2);
            wait_st();
            fence_before();
            mbar_arrive(&S.a2[e]);
            mbar_wait(&S.d2[e], use & 1);
            fence_after();
            uint32_t p0[32], p1[32], p2[32];
            LD32(base + 64, p0);
            LD32(base + 96, p1);
            LD32(base + 128, p2);
            wait_ld();
            fence_before();
            mbar_arrive(&S.fr[e]);
            double h0 = 0.0, h1 = 0.0;
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const int32_t c0 = (int32_t)(p0[i] + (p1[i] << 8) + (p2[i] << 16));
                const int32_t c1 = (int32_t)(p0[i + 1] + (p1[i + 1] << 8) + (p2[i + 1] << 16));
                h0 = fma(S.Wt[i * 32 + k], fabs((double)c0), h0);
                h1 = fma(S.Wt[(i + 1) * 32 + k], fabs((double)c1), h1);
            }
            H += h0 + h1;
            if (t == 0) {  // block b's H of tile 0 (the check)
                double v = h0 + h1;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0 && blockIdx.x == 0) Hout[b] = v;
            }
        }
        if (H == 12345.678) Hout[8] = H;  // keep the epilogue alive
    }
    fence_before();
    __syncthreads();
    if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

// Software-pipelined variant: two epilogue sets, each slot with two A2 plane regions, so a set
// splits tile j + 1 while pass 2 of tile j runs on the tensor core.  Slot (192 columns): D1 [0,32),
// A2[0] [32,56), A2[1] [64,88), D2 [96,192).
constexpr int kSlotP = 192;
__global__ void __launch_bounds__(32 * 9, 1)
k_dct32_pipe(const int8_t *T, const uint8_t *X, const double *W, int tiles, double *Hout)
{
    extern __shared__ __align__(1024) uint8_t dyn[];
    Smem &S = *reinterpret_cast<Smem *>(dyn);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 32 * 128; i += blockDim.x) {
        const int y = i / 128, k = i % 128;
        S.B1[kmaj(y, k, 128, 1024)] = X[(k / 32) * 1024 + y * 32 + (k % 32)];
    }
    for (int i = tid; i < 32 * 32; i += blockDim.x) {
        const int r = i / 32, k = i % 32;
        S.B2[kmaj(r, k, 128, 256)] = (uint8_t)T[r * 32 + k];
        S.Wt[i] = W[i];
    }
    if (tid == 0) {
        for (int e = 0; e < 2; ++e) {
            mbar_init(&S.d1[e], 1);
            mbar_init(&S.a2[e], 128);
            mbar_init(&S.d2[e], 1);
            mbar_init(&S.fr[e], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&S.tbase))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = S.tbase;
    if (warp >= 1 && warp <= 4) {
        const int b = warp & 3, k = lane;
        const uint32_t lanebase = tm + ((uint32_t)(32 * b) << 16);
        for (int cb = 0; cb < 4; ++cb) {
            uint32_t w[8];
            for (int c = 0; c < 8; ++c) {
                uint32_t v = 0;
                for (int q = 0; q < 4; ++q) {
                    const int kk = cb * 32 + 4 * c + q;
                    const int t = kk / 32 == b ? (int)T[k * 32 + kk % 32] : 0;
                    v |= (uint32_t)(t & 255) << (8 * q);
                }
                w[c] = v;
            }
            ST8(lanebase + 8 * cb, w);
        }
        wait_st();
    }
    fence_before();
    __syncthreads();
    fence_after();
    const int nj0 = (tiles + 1) / 2, nj1 = tiles / 2;  // tiles of set 0 (even) and set 1 (odd)
    if (warp == 0) {
        if (lane == 0) {
            const uint32_t id1 = idesc_i8(128, 32, true, false);
            const uint64_t b1 = sdesc(smem_u32(S.B1), 128, 1024);
            const uint64_t b2 = sdesc(smem_u32(S.B2), 128, 256);
            auto pass1 = [&](int e) {
                const uint32_t D1 = tm + 32 + e * kSlotP;
#pragma unroll
                for (int kb = 0; kb < 4; ++kb) mma_ts(D1, tm + 8 * kb, b1 + (uint64_t)(kb * 16), id1, kb);
                commit(&S.d1[e]);
            };
            if (nj0 > 0) pass1(0);
            if (nj1 > 0) pass1(1);
            for (int r = 0; r < nj0; ++r)
                for (int e = 0; e < 2; ++e) {
                    const int nj = e ? nj1 : nj0;
                    if (r >= nj) continue;
                    mbar_wait(&S.a2[e], r & 1);                      // split(r) done: D1 consumed
                    if (r > 0) mbar_wait(&S.fr[e], (r - 1) & 1);     // D2(r - 1) loaded
                    fence_after();
                    const uint32_t base = tm + 32 + e * kSlotP;
                    const uint32_t A2 = base + 32 + 32 * (r & 1), D2 = base + 64 + 32;
#pragma unroll
                    for (int p = 0; p < 3; ++p) mma_ts(D2 + 32 * p, A2 + 8 * p, b2, idesc_i8(128, 32, p == 2, true), 0);
                    commit(&S.d2[e]);
                    if (r + 1 < nj) pass1(e);
                }
        }
    } else {
        const int e = (warp - 1) >> 2, b = warp & 3, k = lane;
        const uint32_t base = tm + ((uint32_t)(32 * b) << 16) + 32 + e * kSlotP;
        const int nj = e ? nj1 : nj0;
        auto split = [&](int j) {
            mbar_wait(&S.d1[e], j & 1);
            fence_after();
            uint32_t z[32];
            LD32(base, z);
            wait_ld();
            uint32_t w0[8], w1[8], w2[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint32_t v0 = z[4 * c], v1 = z[4 * c + 1], v2 = z[4 * c + 2], v3 = z[4 * c + 3];
                const uint32_t s0 = __byte_perm(v0, v1, 0x5140), s1 = __byte_perm(v0, v1, 0x7362);
                const uint32_t s2 = __byte_perm(v2, v3, 0x5140), s3 = __byte_perm(v2, v3, 0x7362);
                w0[c] = __byte_perm(s0, s2, 0x5410);
                w1[c] = __byte_perm(s0, s2, 0x7632);
                w2[c] = __byte_perm(s1, s3, 0x5410);
            }
            const uint32_t A2 = base + 32 + 32 * (j & 1);
            ST8(A2, w0);
            ST8(A2 + 8, w1);
            ST8(A2 + 16, w2);
            wait_st();
            fence_before();
            mbar_arrive(&S.a2[e]);
        };
        double H = 0.0;
        if (nj > 0) split(0);
        for (int j = 0; j < nj; ++j) {
            if (j + 1 < nj) split(j + 1);  // overlaps pass 2 of tile j
            mbar_wait(&S.d2[e], j & 1);
            fence_after();
            uint32_t p0[32], p1[32], p2[32];
            LD32(base + 96, p0);
            LD32(base + 128, p1);
            LD32(base + 160, p2);
            wait_ld();
            fence_before();
            mbar_arrive(&S.fr[e]);
            double h0 = 0.0, h1 = 0.0;
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const int32_t c0 = (int32_t)(p0[i] + (p1[i] << 8) + (p2[i] << 16));
                const int32_t c1 = (int32_t)(p0[i + 1] + (p1[i + 1] << 8) + (p2[i + 1] << 16));
                h0 = fma(S.Wt[i * 32 + k], fabs((double)c0), h0);
                h1 = fma(S.Wt[(i + 1) * 32 + k], fabs((double)c1), h1);
            }
            H += h0 + h1;
            if (j == 0 && e == 0) {
                double v = h0 + h1;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0 && blockIdx.x == 0) Hout[b] = v;
            }
        }
        if (H == 12345.678) Hout[8] = H;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

int main()
{
    setvbuf(stdout, NULL, _IONBF, 0);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    // basis T (R-1), weights w(i,k) / (4096 n) (DC excluded), pixels of 4 blocks
    std::vector<int8_t> T(32 * 32);
    for (int k = 0; k < 32; ++k)
        for (int x = 0; x < 32; ++x) {
            const double ck = k == 0 ? std::sqrt(0.5) : 1.0;
            T[k * 32 + x] = (int8_t)std::lround(64.0 * std::sqrt(2.0) * ck * std::cos(M_PI * (2 * x + 1) * k / 64.0));
        }
    std::vector<double> W(32 * 32);
    for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 32; ++j) {
            const double r = (double)(i * j) / 1024.0;
            W[i * 32 + j] = (i == 0 && j == 0) ? 0.0 : std::exp(std::fabs(r * r - 1.0)) / (4096.0 * 32);
        }
    std::vector<uint8_t> X(4 * 1024);
    srand(7);
    for (auto &v : X) v = (uint8_t)(rand() & 255);
    // host reference: H of each block, exact integer DCT (C[i][j] = sum_yx T[i][y] T[j][x] X[y][x])
    double Href[4];
    for (int b = 0; b < 4; ++b) {
        double acc = 0.0;
        for (int i = 0; i < 32; ++i)
            for (int j = 0; j < 32; ++j) {
                int64_t c = 0;
                for (int y = 0; y < 32; ++y) {
                    int64_t zz = 0;
                    for (int x = 0; x < 32; ++x) zz += (int64_t)T[j * 32 + x] * X[b * 1024 + y * 32 + x];
                    c += (int64_t)T[i * 32 + y] * zz;
                }
                acc += W[i * 32 + j] * (double)(c < 0 ? -c : c);
            }
        Href[b] = acc;
    }
    int8_t *dT;
    uint8_t *dX;
    double *dW, *dH;
    long long *dc;
    CK(cudaMalloc(&dT, T.size()));
    CK(cudaMalloc(&dX, X.size()));
    CK(cudaMalloc(&dW, W.size() * 8));
    CK(cudaMalloc(&dH, 16 * 8));
    CK(cudaMalloc(&dc, sms * 8));
    CK(cudaMemcpy(dT, T.data(), T.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dX, X.data(), X.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dW, W.data(), W.size() * 8, cudaMemcpyHostToDevice));
    const int smem = sizeof(Smem) + 1024;
    CK(cudaFuncSetAttribute(k_dct32, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int tiles = 3000;
    const int threads = 32 * (1 + 4 * NSETS);
    k_dct32<<<sms, threads, smem>>>(dT, dX, dW, 8, dH, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    double Hg[4];
    CK(cudaMemcpy(Hg, dH, 32, cudaMemcpyDeviceToHost));
    bool ok = true;
    for (int b = 0; b < 4; ++b) {
        const double rel = std::fabs(Hg[b] - Href[b]) / Href[b];
        printf("block %d: H gpu %.12g host %.12g rel %.2e\n", b, Hg[b], Href[b], rel);
        ok &= rel < 1e-12;
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    k_dct32<<<sms, threads, smem>>>(dT, dX, dW, tiles, dH, dc);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double units = 4.0 * tiles * sms;
    printf("tcgen05 luma-only n=32 pipeline (NSETS=%d, %d epilogue warps): %s; %.3f ms for %.0f luma units = %.3f G units/s"
           " (%.1f SM-cycles per unit at 1.965 GHz)\n",
           NSETS, 4 * NSETS, ok ? "H exact to 1e-12" : "H MISMATCH", ms, units, units / ms / 1e6,
           ms * 1e-3 * 1.965e9 * sms / units);
    // software-pipelined variant
    CK(cudaFuncSetAttribute(k_dct32_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaMemset(dH, 0, 16 * 8));
    k_dct32_pipe<<<sms, 32 * 9, smem>>>(dT, dX, dW, 8, dH);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(Hg, dH, 32, cudaMemcpyDeviceToHost));
    bool ok2 = true;
    for (int b = 0; b < 4; ++b) ok2 &= std::fabs(Hg[b] - Href[b]) / Href[b] < 1e-12;
    CK(cudaEventRecord(e0));
    k_dct32_pipe<<<sms, 32 * 9, smem>>>(dT, dX, dW, tiles, dH);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("tcgen05 luma-only n=32 pipeline, split of tile j+1 under pass 2 of tile j (2 sets, 8 epilogue warps): %s; "
           "%.3f ms = %.3f G units/s (%.1f SM-cycles per unit)\n",
           ok2 ? "H exact to 1e-12" : "H MISMATCH", ms, units / ms / 1e6, ms * 1e-3 * 1.965e9 * sms / units);
    return ok && ok2 ? 0 : 1;
}
