// tcgen05 probe on B200 (sm_100a), for the NEXT-1 design decision (a tcgen05.mma.kind::i8 path for
// the n = 32 DCT family):
//   1. correctness of hand-built descriptors: D[128][N] = A[128][32] . B[32][N] (kind::i8, s32
//      accumulate in TMEM), A K-major or MN-major, B K-major, no swizzle, vs a host reference;
//   2. MMA issue rate: cycles per tcgen05.mma (M = 128, K = 32, N = 32..256), one issuing thread;
//   3. TMEM -> register bandwidth: bytes per SM-cycle of tcgen05.ld.32x32b.x{16,32,64} with
//      4 / 8 / 16 warps (the epilogue of an exact 3-byte-plane pass 2 reads 12 B per coefficient).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc05 tc05.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// tcgen05 shared-memory matrix descriptor, no swizzle (version 1 = sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// instruction descriptor, kind::i8 (s32 accumulate)
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_s8, bool b_s8, bool a_mn, bool b_mn)
{
    return (2u << 4) | ((a_s8 ? 1u : 0u) << 7) | ((b_s8 ? 1u : 0u) << 10) | ((a_mn ? 1u : 0u) << 15) |
           ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
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

__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols) : "memory");
}

#define LD32(addr, r)                                                                                              \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"  \
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                       \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),      \
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),      \
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                            \
                 : "r"(addr))
#define LD16(addr, r)                                                                                              \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"  \
                 " [%16];"                                                                                          \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                   "=r"(r[15])                                                                                      \
                 : "r"(addr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// canonical no-swizzle layouts for 8-bit elements (16-byte core-matrix rows)
// K-major [rows][K]: core (r/8, k/16) at (r/8)*SBO + (k/16)*LBO, inside (r%8)*16 + k%16
__host__ __device__ inline int kmaj(int r, int k, int lbo, int sbo) { return (r / 8) * sbo + (k / 16) * lbo + (r % 8) * 16 + (k % 16); }
// MN-major: core (m/16, k/8) at (m/16)*SBO + (k/8)*LBO, inside (k%8)*16 + m%16
__host__ __device__ inline int mnmaj(int m, int k, int lbo, int sbo) { return (m / 16) * sbo + (k / 8) * lbo + (k % 8) * 16 + (m % 16); }

// ---- 1. correctness: D = A (128 x 32) . B (32 x N), B given as Bt[N][32]
template <int N>
__global__ void k_correct(const int8_t *A, const int8_t *Bt, int a_mn, int a_s8, int b_s8, int32_t *D)
{
    __shared__ __align__(1024) uint8_t sA[128 * 32];
    __shared__ __align__(1024) uint8_t sB[N * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // A: K-major LBO = 128, SBO = 256; MN-major LBO (K groups) = 1024, SBO (M groups) = 128
    for (int i = tid; i < 128 * 32; i += blockDim.x) {
        const int m = i / 32, k = i % 32;
        const int off = a_mn ? mnmaj(m, k, 1024, 128) : kmaj(m, k, 128, 256);
        sA[off] = (uint8_t)A[i];
    }
    for (int i = tid; i < N * 32; i += blockDim.x) {
        const int n = i / 32, k = i % 32;
        sB[kmaj(n, k, 128, 256)] = (uint8_t)Bt[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&tbase, 256);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = tbase;
    if (tid == 0) {
        const uint64_t ad = a_mn ? sdesc(smem_u32(sA), 1024, 128) : sdesc(smem_u32(sA), 128, 256);
        const uint64_t bd = sdesc(smem_u32(sB), 128, 256);
        mma_i8(tm, ad, bd, idesc_i8(128, N, a_s8, b_s8, a_mn, false), 0);
        mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    fence_after();
    for (int c = 0; c < N; c += 32) {
        uint32_t r[32];
        LD32(tm + ((uint32_t)(32 * warp) << 16) + c, r);
        tmem_wait_ld();
        for (int j = 0; j < 32 && c + j < N; ++j) D[(32 * warp + lane) * N + c + j] = (int32_t)r[j];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 256);
}

// ---- 2. MMA issue rate
template <int N, int NACC>
__global__ void k_mma_rate(int iters, long long *cycles)
{
    __shared__ __align__(1024) uint8_t sA[128 * 32];
    __shared__ __align__(1024) uint8_t sB[256 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 32; i += blockDim.x) sA[i] = (uint8_t)(i * 7);
    for (int i = tid; i < 256 * 32; i += blockDim.x) sB[i] = (uint8_t)(i * 3);
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&tbase, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = tbase;
    if (tid == 0) {
        const uint64_t ad = sdesc(smem_u32(sA), 128, 256);
        const uint64_t bd = sdesc(smem_u32(sB), 128, 256);
        const uint32_t id = idesc_i8(128, N, true, false, false, false);
        // warm-up
        for (int i = 0; i < 8; ++i) mma_i8(tm + ((i % NACC) * N) % 512, ad, bd, id, 1);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) mma_i8(tm + ((i % NACC) * N) % 512, ad, bd, id, i >= NACC);
        mma_commit(&bar);
        mbar_wait(&bar, 1);
        const long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 512);
}

// ---- 3. TMEM load bandwidth: every warp loads its lane quadrant, X columns per instruction
template <int X, int DEPTH>
__global__ void k_ld_rate(int iters, long long *cycles, uint32_t *sink)
{
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&tbase, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += DEPTH) {
        uint32_t r[DEPTH][32];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
            const uint32_t col = (uint32_t)(((i + d) * X + (warp >> 2) * 64) & 511);
            if (X == 32) {
                LD32(tm + col, r[d]);
            } else {
                LD16(tm + col, r[d]);
            }
        }
        tmem_wait_ld();
#pragma unroll
        for (int d = 0; d < DEPTH; ++d)
#pragma unroll
            for (int j = 0; j < X; ++j) acc += r[d][j];
    }
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345u) sink[tid] = acc;
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
}

// ---- 1b. TS mode: A (128 x 32 bytes) written into TMEM with tcgen05.st (thread m = lane m, word c =
// K bytes 4c..4c+3, little endian), B from shared memory (K-major, no swizzle), D = A . B in TMEM
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

template <int N>
__global__ void k_correct_ts(const int8_t *A, const int8_t *Bt, int a_s8, int b_s8, int32_t *D, long long *cyc)
{
    __shared__ __align__(1024) uint8_t sB[N * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < N * 32; i += blockDim.x) {
        const int n = i / 32, k = i % 32;
        sB[kmaj(n, k, 128, 256)] = (uint8_t)Bt[i];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&tbase, 256);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = tbase;
    // A row m = 32 warp + lane into TMEM columns [128, 136)
    {
        uint32_t w[8];
        const uint8_t *row = reinterpret_cast<const uint8_t *>(A) + (32 * warp + lane) * 32;
        for (int c = 0; c < 8; ++c)
            w[c] = (uint32_t)row[4 * c] | ((uint32_t)row[4 * c + 1] << 8) | ((uint32_t)row[4 * c + 2] << 16) |
                   ((uint32_t)row[4 * c + 3] << 24);
        const uint32_t ta = tm + ((uint32_t)(32 * warp) << 16) + 128;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(w[0]),
                     "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
        const uint64_t bd = sdesc(smem_u32(sB), 128, 256);
        const uint32_t id = idesc_i8(128, N, a_s8, b_s8, false, false);
        mma_i8_ts(tm, tm + 128, bd, id, 0);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        // rate: 256 dependent-free TS MMAs into 4 accumulators
        const long long t0 = clock64();
        for (int i = 0; i < 256; ++i) mma_i8_ts(tm + 160 + (i & 1) * 32, tm + 128, bd, id, 1);
        mma_commit(&bar);
        mbar_wait(&bar, 1);
        cyc[0] = clock64() - t0;
    }
    fence_before();
    __syncthreads();  // thread 0 has seen both MMA phases complete
    fence_after();
    for (int c = 0; c < N; c += 32) {
        uint32_t r[32];
        LD32(tm + ((uint32_t)(32 * warp) << 16) + c, r);
        tmem_wait_ld();
        for (int j = 0; j < 32 && c + j < N; ++j) D[(32 * warp + lane) * N + c + j] = (int32_t)r[j];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, 256);
}

template <int N>
bool run_correct_ts(int a_s8, int b_s8)
{
    std::vector<int8_t> A(128 * 32), Bt(N * 32);
    srand(777 + N);
    for (auto &v : A) v = (int8_t)(rand() & 255);
    for (auto &v : Bt) v = (int8_t)(rand() & 255);
    int8_t *dA, *dB;
    int32_t *dD;
    long long *dc;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, Bt.size()));
    CK(cudaMalloc(&dD, 128 * N * 4));
    CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, Bt.data(), Bt.size(), cudaMemcpyHostToDevice));
    k_correct_ts<N><<<1, 128>>>(dA, dB, a_s8, b_s8, dD, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> D(128 * N);
    long long cyc = 0;
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            int64_t s = 0;
            for (int k = 0; k < 32; ++k) {
                const int a = a_s8 ? (int)A[m * 32 + k] : (int)(uint8_t)A[m * 32 + k];
                const int b = b_s8 ? (int)Bt[n * 32 + k] : (int)(uint8_t)Bt[n * 32 + k];
                s += a * b;
            }
            if ((int32_t)s != D[m * N + n]) {
                if (bad < 4) printf("  mismatch m=%d n=%d got %d want %lld\n", m, n, D[m * N + n], (long long)s);
                ++bad;
            }
        }
    printf("correct TS (A in TMEM via tcgen05.st) N=%d A %s, B %s: %s (%d bad); %.1f cycles per TS MMA (1 CTA)\n", N,
           a_s8 ? "s8" : "u8", b_s8 ? "s8" : "u8", bad ? "FAIL" : "ok", bad, cyc / 256.0);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    cudaFree(dc);
    return bad == 0;
}

template <int N>
bool run_correct(int a_mn, int a_s8, int b_s8)
{
    std::vector<int8_t> A(128 * 32), Bt(N * 32);
    srand(12345 + N + 7 * a_mn + 3 * a_s8);
    for (auto &v : A) v = (int8_t)(rand() & 255);
    for (auto &v : Bt) v = (int8_t)(rand() & 255);
    int8_t *dA, *dB;
    int32_t *dD;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, Bt.size()));
    CK(cudaMalloc(&dD, 128 * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, Bt.data(), Bt.size(), cudaMemcpyHostToDevice));
    k_correct<N><<<1, 128>>>(dA, dB, a_mn, a_s8, b_s8, dD);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> D(128 * N);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            int64_t s = 0;
            for (int k = 0; k < 32; ++k) {
                const int a = a_s8 ? (int)A[m * 32 + k] : (int)(uint8_t)A[m * 32 + k];
                const int b = b_s8 ? (int)Bt[n * 32 + k] : (int)(uint8_t)Bt[n * 32 + k];
                s += a * b;
            }
            if ((int32_t)s != D[m * N + n]) {
                if (bad < 4) printf("  mismatch m=%d n=%d got %d want %lld\n", m, n, D[m * N + n], (long long)s);
                ++bad;
            }
        }
    printf("correct N=%d A %s %s, B %s: %s (%d bad)\n", N, a_mn ? "MN-major" : "K-major", a_s8 ? "s8" : "u8",
           b_s8 ? "s8" : "u8", bad ? "FAIL" : "ok", bad);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    return bad == 0;
}

template <int N, int NACC>
void run_mma_rate(int sms)
{
    long long *dc;
    CK(cudaMalloc(&dc, sizeof(long long) * sms));
    const int iters = 4096;
    k_mma_rate<N, NACC><<<sms, 128>>>(iters, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(sms);
    CK(cudaMemcpy(c.data(), dc, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
    double mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    const double cyc = mx / iters;
    printf("mma M=128 N=%3d K=32 i8, %d accumulators: %.2f cycles/MMA per SM (%d CTAs), %.0f MACs/cycle/SM\n", N,
           NACC, cyc, sms, 128.0 * N * 32 / cyc);
    cudaFree(dc);
}

template <int X, int DEPTH>
void run_ld_rate(int warps, int sms)
{
    long long *dc;
    uint32_t *sink;
    CK(cudaMalloc(&dc, sizeof(long long) * sms));
    CK(cudaMalloc(&sink, 4 * 1024));
    const int iters = 2048;
    k_ld_rate<X, DEPTH><<<sms, 32 * warps>>>(iters, dc, sink);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<long long> c(sms);
    CK(cudaMemcpy(c.data(), dc, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
    double mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    const double bytes = (double)warps * iters * 32 * X * 4;
    printf("tcgen05.ld 32x32b.x%d, %d in flight, %2d warps/SM: %.1f bytes/cycle/SM (%.1f cycles per warp-load)\n", X,
           DEPTH, warps, bytes / mx, mx / iters);
    cudaFree(dc);
    cudaFree(sink);
}

int main()
{
    setvbuf(stdout, NULL, _IONBF, 0);
    int dev = 0, sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    bool ok = true;
    ok &= run_correct<32>(0, 1, 0);   // A s8 K-major, B u8
    ok &= run_correct<32>(0, 0, 1);   // A u8 K-major, B s8 (pixels x basis)
    ok &= run_correct<32>(1, 0, 1);   // A u8 MN-major (pixel columns), B s8
    ok &= run_correct<64>(0, 1, 0);
    ok &= run_correct<16>(0, 0, 1);
    ok &= run_correct<32>(1, 1, 1);
    ok &= run_correct_ts<32>(1, 0);
    ok &= run_correct_ts<32>(0, 1);
    printf("descriptor correctness: %s\n", ok ? "all ok" : "FAILURES");
    run_mma_rate<32, 2>(sms);
    run_mma_rate<32, 8>(sms);
    run_mma_rate<32, 16>(sms);
    run_mma_rate<64, 2>(sms);
    run_mma_rate<64, 8>(sms);
    run_mma_rate<128, 2>(sms);
    run_mma_rate<128, 4>(sms);
    run_mma_rate<256, 2>(sms);
    for (int w : {4, 8, 16}) {
        run_ld_rate<32, 1>(w, sms);
        run_ld_rate<32, 2>(w, sms);
        run_ld_rate<32, 4>(w, sms);
        run_ld_rate<16, 4>(w, sms);
    }
    return 0;
}
