// Microbenchmark: per-SM throughput of the epilogue instruction candidates on B200
// (I2F.F64, DFMA, IMAD.WIDE, IDP.4A, PRMT, F2F) -- warp-instructions per SM-cycle.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N_IT 4096
template <int K>
__global__ void kern(int32_t *out, int seed, long long *cyc)
{
    int32_t a[8];
    double d[8];
    uint64_t w[8];
    float f[8];
    for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 7 + i; d[i] = a[i]; w[i] = a[i]; f[i] = a[i]; }
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (K == 0) { double x; asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(x) : "r"(a[i])); d[i] = fma(d[i], 1.0000001, x); a[i] = __double2loint(d[i]); }  // I2F.F64 + DFMA
            if (K == 1) d[i] = fma(d[i], 1.0000001, d[(i + 1) & 7]);                      // DFMA only
            if (K == 2) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[i]) : "r"(a[i]), "r"((uint32_t)w[(i + 3) & 7]));  // IMAD.WIDE.U32
            if (K == 3) a[i] = __dp4a(a[i], 0x40404040, a[(i + 1) & 7]);                 // IDP.4A
            if (K == 4) a[i] = __byte_perm(a[i], a[(i + 1) & 7], 0x5140);                 // PRMT
            if (K == 5) d[i] += (double)f[i] , f[i] += 1.0f;                              // F2F.F64.F32 + DADD + FADD
            if (K == 6) a[i] = a[i] * 0x01000193 + a[(i + 1) & 7];                        // IMAD
            if (K == 7) { asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(d[i]) : "r"(a[i])); a[i] = __double2hiint(d[i]); }  // I2F.F64 (chained)
        }
    }
    long long t1 = clock64();
    int32_t s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + (int)d[i] + (int)w[i] + (int)(w[i] >> 32) + (int)f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int K>
void run(const char *name, int32_t *out, long long *cyc)
{
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 512, blocks = nsm * 2;
    kern<K><<<blocks, threads>>>(out, 1, cyc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<K><<<blocks, threads>>>(out, 1, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double warp_instr = (double)blocks * threads / 32 * N_IT * 8;  // of the "main" op
    double per_sm_cycle = warp_instr / nsm / (double)c;
    printf("%-28s %8.3f ms  cycles(block0)=%lld  main warp-ops per SM-cycle = %.3f (lanes/clk/SM = %.1f)\n", name, ms,
           c, per_sm_cycle, per_sm_cycle * 32);
}

int main()
{
    int32_t *out; long long *cyc;
    cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
    run<0>("I2F.F64+DFMA", out, cyc);
    run<1>("DFMA", out, cyc);
    run<2>("IMAD.WIDE.U32", out, cyc);
    run<3>("IDP.4A", out, cyc);
    run<4>("PRMT", out, cyc);
    run<5>("F2F.F64.F32+DADD+FADD", out, cyc);
    run<6>("IMAD", out, cyc);
    run<7>("I2F.F64 (+IADD)", out, cyc);
    return 0;
}
