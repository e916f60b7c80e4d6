// Read-only HBM streaming bandwidth on B200 (context for the block kernel's roofline, which
// reads its frames once and writes ~1 %): each thread sums 16-byte vectors of a 7.5 GB
// buffer (larger than L2), grid = SMs x k CTAs; best of 10, CUDA events.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) read_kernel(const uint4 *__restrict__ p, size_t n, unsigned *out)
{
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 4
    for (; i < n; i += stride) {
        const uint4 v = __ldcs(p + i);  // streaming (evict-first) load
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;  // keep the loads alive
}

int main()
{
    const size_t bytes = (size_t)7464960000ull;  // config 3: 600 UHD 8-bit frames
    const size_t n = bytes / sizeof(uint4);
    uint4 *p;
    unsigned *out;
    if (cudaMalloc(&p, bytes) != cudaSuccess || cudaMalloc(&out, 4) != cudaSuccess) return 1;
    cudaMemset(p, 1, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int k : {2, 4, 8}) {
        float best = 1e30f;
        for (int rep = 0; rep < 10; ++rep) {
            cudaEventRecord(e0);
            read_kernel<<<sms * k, 512>>>(p, n, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("read-only stream, grid %d x 512: %.1f GB/s (best of 10)\n", sms * k, bytes / (best / 1e3) / 1e9);
    }
    return 0;
}
