// vca_common.cuh -- shared device-side definitions of libvca (product path).
// Citations: P:n = PAPER.md, S:n = SPEC.md, R-k = DESIGN.md readings.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vca {

// Offsets of the per-size tables inside the concatenated device arrays:
// basis T_n (int8, n*n) and scaled weights wts_n(i,j) = w_n(i,j)/(4096 n)
// (double, n*n, 0 at (0,0)), for n = 4, 8, 16, 32.
__host__ __device__ constexpr int table_offset(int n)
{
    return n == 4 ? 0 : n == 8 ? 16 : n == 16 ? 80 : 336;
}
constexpr int kTableElems = 16 + 64 + 256 + 1024;

// Kernel parameters of one analysis call (all device pointers).
struct PlaneDesc {
    const uint8_t *base;  // frame 0, row 0
    int64_t pitch;        // bytes between rows
    int64_t fstride;      // bytes between frames
    int width, height;    // samples
    int w;                // block size in samples
    int n;                // DCT size (w or w/2)
    int cols, rows;       // block grid
    int64_t count;        // cols * rows
};

struct Scratch {
    double *HY;        // [n_frames][C_Y] per-block luma texture energy (A5), raster order
    double *partial;   // [n_frames][3][P][2]: (sum H, sum L) partial sums, fixed order (A7)
    int P;             // partial entries per plane (stride)
    int Pp[3];         // partial entries used by plane p
};

}  // namespace vca
