// kernel_fused.cuh -- the fused hot-path kernel (A1-A7) for every block configuration
// whose chroma grid equals the luma grid: luma block w in {8, 16, 32} (n = 32, 16, 8
// families; low-pass needs w >= 16), chroma block w/2, 8- or 10-bit.  w = 4 (chroma grid
// half the luma grid) runs small_block_kernel in kernel_generic.cuh.
//
// One work item = one block row r of one frame f; a unit = the co-located Y block
// (w x w) and U, V blocks (w/2 x w/2) of (f, r, c); a strip = 4 * NU consecutive units.
// One persistent CTA per SM, warp-specialised (3 consumer groups; 4 for the n = 8 families):
//
//  * warpgroup 0: producers (setmaxnreg.dec).  Warp g's elected lane feeds consumer
//    group g: per strip one 4-D tensor-map load per plane (all of the strip's boxes; 3-D
//    loads per box where the geometry does not allow it), swizzled, zero-filled out of
//    bounds, into the group's ring of smem stages, full/empty mbarriers (A1);
//  * warpgroups 1..G: consumer groups of 4 warps (setmaxnreg.inc), each walking its own
//    item sequence; warp u owns units u + 4n (n < NU) of every strip.  A consumer reads
//    its units from smem with clamped row/column indices (edge replication, A2),
//    low-pass-downsamples in registers with (s+2)>>2 (A3, R-5), and runs the exact
//    integer DCT C = T X T^T on the tensor cores (A4, R-1) as two passes that never
//    leave registers:
//        pass 1   Z^T = T . X^T      (s8 basis x u8 pixels -> s32; 10-bit n = 16/8:
//                                     f16 x f16 -> f32 with an exact magic offset)
//        pass 2   C   = T' . Z'      with Z split in three byte planes
//                 (u8, u8, s8) and C = D0 + 2^8 D1 + 2^16 D2 (mod 2^32);
//    the C-fragment layout of pass 1 is, up to a fixed permutation pi of the
//    contraction index y, the B-fragment layout of pass 2, so T' = T[:, pi]
//    (a constant) absorbs the transpose -- no shuffles, no smem round trip.
//    Chroma 8x8 DCTs pair U and V block-diagonally into one 16x16 MMA.
//  * the epilogue (A5, A6, R-2, R-3): luma |C_ij| x w_n(i,j)/(4096 n) in FP64 per
//    block (needed per block for h), chroma |C| summed exactly per coefficient
//    position in uint32 and weighted once per flush; per-(frame, row, warp) partial
//    sums in a fixed order (A7 inputs, R-11), the six per-lane running sums reduced across
//    the warp once per item by one reduce-scatter (xred8).  The finalize kernel
//    (kernel_finalize.cuh) turns the partials and the per-block H_Y into records (A7-A9).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include <atomic>

#include "kernel_generic.cuh"
#include "vca_common.cuh"

namespace vca {

// A/B (tools/ab_variants.py, 600 frames): G = 3 groups with 152-register consumers and
// NU = 4 units per warp per strip: config 3 400k -> 432k fps, config 2 545k -> 565k, config 4
// flat; G = 4 (104 registers) or G = 2 (8 consumer warps) are slower.
#ifndef VCA_GROUPS
#define VCA_GROUPS 3
#endif

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

#ifndef VCA_WAIT_HINT
#define VCA_WAIT_HINT 1000000
#endif
// Blocking wait on an mbarrier phase; the suspend-time hint lets the warp sleep
// in try_wait until the phase completes instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "VCA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra VCA_WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity), "r"(VCA_WAIT_HINT)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y, int z,
                                            uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// One 4-D tensor-map load of a strip's NB boxes of a plane (dims: bytes within a box row, rows,
// box index along the row, frame): the same smem layout as NB 3-D box loads, one TMA instruction
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c, int y, int z,
                                            uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(y), "r"(c), "r"(z), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// Stores of the per-block H_Y and the per-row partials that the finalize kernel reads right
// after this kernel: with VCA_EVICT_LAST they carry an L2 evict_last hint (the frames stream
// through L2 evict_first), so the finalize reads them from L2.  A/B: block kernel -1.4 %,
// finalize unchanged (profiles/r02/ab_evict_last_reverted.log); off.
#ifndef VCA_EVICT_LAST
#define VCA_EVICT_LAST 0
#endif
__device__ __forceinline__ void st_keep(double *p, double v, uint64_t pol)
{
#if VCA_EVICT_LAST
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
    (void)pol;
    *p = v;
#endif
}

#ifndef VCA_TMA4
#define VCA_TMA4 1  // use the 4-D maps where the plane geometry allows (A/B: 0 = always 3-D)
#endif

// L2 prefetch of a box a few strips ahead of the ring (VCA_L2PF strips; 0 = off): the later
// TMA load of the same box then hits L2 instead of HBM.  A/B (profiles/r02/ab_l2_prefetch_reverted.log,
// 1 / 2 / 4 strips ahead): config 3 -4 %, config 4 -2..-4 %, config 2 -2 % -- off.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *map, int x, int y, int z)
{
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(z)
                 : "memory");
}
#ifndef VCA_L2PF
#define VCA_L2PF 0
#endif

#define VCA_MMA_ASM asm volatile  // A/B: non-volatile (reorderable) MMA asm was neutral
// D = A(s8) . B(u8) + C, m16n8k16
__device__ __forceinline__ void mma16_su(int32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t b)
{
    VCA_MMA_ASM("mma.sync.aligned.m16n8k16.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%7,%8,%9,%10};"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
                 : "r"(a0), "r"(a1), "r"(b), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void mma16_ss(int32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t b)
{
    VCA_MMA_ASM("mma.sync.aligned.m16n8k16.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%7,%8,%9,%10};"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
                 : "r"(a0), "r"(a1), "r"(b), "r"(0), "r"(0), "r"(0), "r"(0));
}
// m16n8k32
__device__ __forceinline__ void mma32_su(int32_t (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1)
{
    VCA_MMA_ASM(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%12,%13};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void mma32_ss(int32_t (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1)
{
    VCA_MMA_ASM(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%12,%13};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(0), "r"(0), "r"(0), "r"(0));
}

// D = A(u8) . B(u8) + C, m16n8k32 (the 2x2 low-pass sums, C = rounding offset)
__device__ __forceinline__ void mma32_uu_acc(int32_t (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                             const int32_t (&c)[4])
{
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%12,%13};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]));
}

// D = A(f16) . B(f16) + C (f32), m16n8k16 -- the exact 10-bit pass 1 (see dct16h)
__device__ __forceinline__ void mma16_h(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1, float c)
{
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%10,%10,%10};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c));
}
// D = A(f16) . B(f16) + C (f32, per element), m16n8k16 -- the 8-bit two-plane pass 2
__device__ __forceinline__ void mma16_hc(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1, float c0, float c1, float c2, float c3)
{
    VCA_MMA_ASM(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%12,%13};"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(c0), "f"(c1), "f"(c2), "f"(c3));
}
// pass 2 with a per-lane accumulator init (the corrections of the 10-bit path)
__device__ __forceinline__ void mma16_su_c(int32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t b, int32_t c0,
                                           int32_t c1, int32_t c2, int32_t c3)
{
    VCA_MMA_ASM("mma.sync.aligned.m16n8k16.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%7,%8,%9,%10};"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
                 : "r"(a0), "r"(a1), "r"(b), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
}

// byte planes b = 0, 1, 2 of four int32 values (v0..v3 -> bytes 0..3 of each plane)
__device__ __forceinline__ void byte_planes(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3, uint32_t &p0,
                                            uint32_t &p1, uint32_t &p2)
{
    const uint32_t s0 = __byte_perm(v0, v1, 0x5140);  // v0.b0 v1.b0 v0.b1 v1.b1
    const uint32_t s1 = __byte_perm(v0, v1, 0x7362);  // v0.b2 v1.b2 v0.b3 v1.b3
    const uint32_t s2 = __byte_perm(v2, v3, 0x5140);
    const uint32_t s3 = __byte_perm(v2, v3, 0x7362);
    p0 = __byte_perm(s0, s2, 0x5410);
    p1 = __byte_perm(s0, s2, 0x7632);
    p2 = __byte_perm(s1, s3, 0x5410);
}

// Exact double of an int32 without the conversion pipe (I2F.F64 retires 16 lanes/clk/SM on
// B200, DADD 64; tools/micro/pipes.cu): with M = 2^52 + 2^51, the double M + c has low word c
// and high word 0x43380000 + (c >> 31) (one LEA.HI.SX32), and (M + c) - M = c exactly (DADD).
// A/B (config 2/3/4): I2F.F64 is faster overall -- the kernel is issue-bound, not XU-bound,
// and the magic form costs an extra instruction -- so it is the default.
__device__ __forceinline__ double i2d(int32_t c)
{
#ifndef VCA_CVT_MAGIC
    return __int2double_rn(c);
#else
    return __hiloint2double(0x43380000 + (c >> 31), c) - 6755399441055744.0;
#endif
}

__device__ __forceinline__ int32_t combine3(int32_t d0, int32_t d1, int32_t d2)
{
    return (int32_t)((uint32_t)d0 + ((uint32_t)d1 << 8) + ((uint32_t)d2 << 16));
}

// ------------------------------------------------------------------ family geometry
template <int W_, int BD_, int LP_>
struct Fam {
    static constexpr int W = W_, WC = W_ / 2, BD = BD_, LP = LP_;
    static constexpr int ES = BD == 8 ? 1 : 2;
    static constexpr int NY = LP ? W / 2 : W;
    static constexpr int NC = LP ? WC / 2 : WC;
#ifndef VCA_GROUPS8
#define VCA_GROUPS8 4  // consumer groups of the n = 8 families (A/B: 4 groups of 112 registers, NU8 = 4:
                       // 1080p lp16 +3 %, 1080p w8 +7 %, 720p lp16 +20 %, 720p w8 +-0 vs 3 groups, NU8 = 8)
#endif
    // consumer groups per CTA (0: the legacy one-producer-warp layout), threads per CTA
#ifndef VCA_GROUPS32
#define VCA_GROUPS32 VCA_GROUPS  // consumer groups of the n = 32 families (A/B)
#endif
    static constexpr int G = NY == 8 ? VCA_GROUPS8 : NY == 32 ? VCA_GROUPS32 : VCA_GROUPS;
    static constexpr int GV = G ? G : 1;
    static constexpr int THREADS = G ? 128 * (1 + G) : 160;
    static_assert(G >= 0 && G <= 4, "one producer warp per consumer group, all in warpgroup 0");
#ifndef VCA_NU
#define VCA_NU (VCA_GROUPS == 3 ? 4 : 2)
#endif
#ifndef VCA_STAGE_MAX
#define VCA_STAGE_MAX 24576  // largest n = 16 luma stage (6 NU ES W^2 bytes) before NU falls back to 2
#endif
#ifndef VCA_NU8
// units per warp per strip, n = 8 families (multiple of 4; with 3 groups, A/B: 8 vs 4 +6.5 %
// 1080p lp16, +17 % 720p w8; 4 groups fit only 4 in shared memory)
#define VCA_NU8 (VCA_GROUPS8 >= 4 ? 4 : 8)
#endif
#ifndef VCA_NU32
#define VCA_NU32 2  // units per consumer warp per strip for the n = 32 luma path (A/B: 1 -> 2 +3 %)
#endif
    // units per consumer warp per strip (ILP, per-strip overhead); 4 only while a 16-unit stage
    // stays <= 24 KB (two stages per group, three groups per CTA)
    static constexpr int NU = NY == 32  ? VCA_NU32
                              : NY == 8 ? VCA_NU8  // groups of 4: 2 luma pairs + one 8-block chroma MMA
                              : (6 * VCA_NU * ES * W * W > VCA_STAGE_MAX) ? (VCA_GROUPS == 4 ? 1 : 2) : VCA_NU;
    // (VCA_GROUPS = 4 is an A/B variant only: 16 consumer warps at 112 registers, NU = 3,
    // 2 x 18 KB stages per group -- 3 % slower on config 3, profiles/r01d/ab_groups4.log)
    static constexpr int UNITS = 4 * NU;                   // units per strip (4 consumer warps)
    static constexpr int RB_Y = W * ES, RB_C = WC * ES;    // bytes per unit row
    // box inner bytes = swizzle span: the largest of 128/64/32 bytes that tiles the strip row
    static constexpr int ib(int row) { return row % 128 == 0 ? 128 : row % 64 == 0 ? 64 : 32; }
    static constexpr int IB_Y = ib(UNITS * RB_Y);
    static constexpr int IB_C = ib(UNITS * RB_C);
    static_assert((UNITS * RB_Y) % IB_Y == 0 && (UNITS * RB_C) % IB_C == 0, "boxes tile the strip");
    static constexpr int SPF = 32 / NU;  // strips per stash flush (<= 32 units stashed)
    static constexpr int UPB_Y = IB_Y / RB_Y, UPB_C = IB_C / RB_C;        // units per box
    static constexpr int NBOX_Y = UNITS / UPB_Y, NBOX_C = UNITS / UPB_C;
    // smem stride per box: whole swizzle atoms (8 rows x IB bytes), so every box starts at an
    // atom-aligned address and swz() (relative to the box) matches the TMA's absolute pattern
    // (chroma boxes of the w = 8 family have only 4 rows)
    static constexpr int BOXB_Y = IB_Y * (W < 8 ? 8 : W), BOXB_C = IB_C * (WC < 8 ? 8 : WC);
    static constexpr int ST_Y = NBOX_Y * BOXB_Y, ST_C = NBOX_C * BOXB_C;
    static constexpr int TX = NBOX_Y * IB_Y * W + 2 * NBOX_C * IB_C * WC;   // bytes landing per stage
    static constexpr int STAGE = (ST_Y + 2 * ST_C + 1023) / 1024 * 1024;
#ifndef VCA_RING
#define VCA_RING 55296  // ring bytes per consumer group: 3 x 18 KB (NU = 3), 2 x 24 KB (NU = 4)
#endif
#ifndef VCA_RING16
#define VCA_RING16 VCA_RING  // ring of the n = 16 luma families (A/B of larger strips)
#endif
#ifndef VCA_RING8
#define VCA_RING8 (VCA_GROUPS8 == 4 ? 36864 : VCA_RING)  // ring of the n = 8 families
#endif
#ifndef VCA_RING32
#define VCA_RING32 VCA_RING  // ring of the n = 32 families (A/B)
#endif
    static constexpr int RING = NY == 16 ? VCA_RING16 : NY == 8 ? VCA_RING8 : NY == 32 ? VCA_RING32 : VCA_RING;
    static constexpr int STAGES = (RING / STAGE) < 2 ? 2 : (RING / STAGE > 16 ? 16 : RING / STAGE);
    static constexpr bool WTAB = (NY == 32);
#ifndef VCA_NO_HMMA10
    // 10-bit n = 16 / paired n = 8 pass 1 on f16 tensor cores (one HMMA instead of a lo/hi
    // pair of IMMAs plus their recombination; exact, see dct16h)
    static constexpr bool H10 = (ES == 2) && (NY == 16);
#else
    static constexpr bool H10 = false;
#endif
#ifndef VCA_MINB
#define VCA_MINB 3
#endif
    static constexpr int MINB = VCA_MINB;  // CTAs/SM of the legacy layout (kGroups == 0)
    // per consumer warp: [32 slots][9] doubles (8 luma row-group partials + pad) + [32][4] DC words
    // luma H partials stashed per unit: one per row group (the 4 lanes of a row group reduced by
    // shuffles) or, with VCA_HHALF on the n = 16 luma families, one per half row group (lanes t = 0,
    // 2 after one shuffle round; the flush adds 16 instead of 8)
#ifndef VCA_HHALF
#define VCA_HHALF 1
#endif
    static constexpr int HSLOTS = (VCA_HHALF && NY == 16 && LP) ? 16 : 8;  // (w = 16 full: over the smem limit)
    static constexpr int HW = HSLOTS + 1;  // padded row of the stash
    static constexpr int STASH = 32 * HW * 8 + 32 * 4 * 4;
    static_assert(NC == NY / 2, "chroma DCT is half the luma DCT");
    static_assert(IB_Y == 32 || IB_Y == 64 || IB_Y == 128, "swizzle span");
    static_assert(IB_C == 32 || IB_C == 64 || IB_C == 128, "swizzle span");
};

template <int IB>
__device__ __forceinline__ uint32_t swz(uint32_t off)
{
    constexpr uint32_t m = IB / 16 - 1;   // 128B: bits 4-6 ^= bits 7-9; 64B: 4-5 ^= 7-8; 32B: 4 ^= 7
    return off ^ (((off >> 7) & m) << 4);
}

// Data-path shared-memory accesses take byte OFFSETS into the dynamic shared array and are
// plain C++ loads/stores: the compiler knows the address space (LDS/STS with immediate
// offsets, no generic-window arithmetic) and schedules them freely between the volatile,
// memory-clobbering mbarrier wait and arrive.  Barriers and TMA take shared addresses
// (smem_u32).
extern __shared__ __align__(1024) uint8_t vca_dyn_smem[];
__device__ __forceinline__ uint32_t smem_off(const void *p)
{
    return (uint32_t)(reinterpret_cast<const uint8_t *>(p) - vca_dyn_smem);
}
#ifdef VCA_DEBUG_BOUNDS
// debug builds (tests/test_bounds_gpu.py): every data-path shared access is checked against
// the dynamic shared-memory size and its natural alignment
__device__ __forceinline__ void smem_check(uint32_t off, uint32_t bytes)
{
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (off + bytes > dyn || (off & (bytes - 1)) != 0) {
        printf("VCA_DEBUG_BOUNDS: smem access %u+%u outside [0, %u) or misaligned (block %d thread %d)\n", off, bytes,
               dyn, blockIdx.x, threadIdx.x);
        __trap();
    }
}
#define VCA_SMEM_CHECK(off, T) smem_check(off, sizeof(T))
#else
#define VCA_SMEM_CHECK(off, T) ((void)0)
#endif
template <class T>
__device__ __forceinline__ T lds(uint32_t off)
{
    VCA_SMEM_CHECK(off, T);
    return *reinterpret_cast<const T *>(vca_dyn_smem + off);
}
template <class T>
__device__ __forceinline__ void sts(uint32_t off, T v)
{
    VCA_SMEM_CHECK(off, T);
    *reinterpret_cast<T *>(vca_dyn_smem + off) = v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) { return lds<uint8_t>(a); }
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) { return lds<uint16_t>(a); }
__device__ __forceinline__ uint32_t lds32(uint32_t a) { return lds<uint32_t>(a); }
__device__ __forceinline__ uint2 lds64(uint32_t a) { return lds<uint2>(a); }
__device__ __forceinline__ uint4 lds128(uint32_t a) { return lds<uint4>(a); }
__device__ __forceinline__ double lds_f64(uint32_t a) { return lds<double>(a); }

// One sample of a unit in a swizzled box (row, column within the unit), 10-bit clamp
template <int ES, int IB>
__device__ __forceinline__ int box_sample(uint32_t box, int ub0, int row, int xs)
{
    if (ES == 1) return (int)lds_u8(box + swz<IB>(row * IB + ub0 + xs));
    const int v = (int)lds_u16(box + swz<IB>(row * IB + ub0 + 2 * xs));
    return v < 1023 ? v : 1023;
}

// 8-bit 2x2 low-pass of two source rows of 8 bytes -> 4 packed outputs, (s+2)>>2 (R-5)
// Each 32-bit word holds 4 samples; even/odd samples go to 16-bit lanes (LOP3 /
// PRMT), the 2x2 sums (<= 1020) plus 2 are formed per lane, and the final PRMT
// picks byte 0 of each lane after >> 2 (s >> 2 <= 255, so no masking is needed).
__device__ __forceinline__ uint32_t ds8(uint2 a, uint2 b)
{
    // 2x2 sums as byte dot products on the FMA pipe (IDP.4A) with weights 64: s' = 64 (s + 2)
    // < 2^16, so byte 1 of s' is (s + 2) >> 2 and three PRMTs pack the four outputs
    const uint32_t s0 = __dp4a(a.x, 0x00004040u, __dp4a(b.x, 0x00004040u, 128u));
    const uint32_t s1 = __dp4a(a.x, 0x40400000u, __dp4a(b.x, 0x40400000u, 128u));
    const uint32_t s2 = __dp4a(a.y, 0x00004040u, __dp4a(b.y, 0x00004040u, 128u));
    const uint32_t s3 = __dp4a(a.y, 0x40400000u, __dp4a(b.y, 0x40400000u, 128u));
    return __byte_perm(__byte_perm(s0, s1, 0x0051), __byte_perm(s2, s3, 0x0051), 0x5410);
}

// four (2x2 sum + 2) values < 1024 -> packed bytes (s >> 2): low halves paired by PRMT,
// one shift per pair, byte 0 / byte 2 of each picked by the final PRMT
__device__ __forceinline__ uint32_t pack_ds(int32_t s0, int32_t s1, int32_t s2, int32_t s3)
{
    const uint32_t t01 = __byte_perm((uint32_t)s0, (uint32_t)s1, 0x5410);
    const uint32_t t23 = __byte_perm((uint32_t)s2, (uint32_t)s3, 0x5410);
    return __byte_perm(t01 >> 2, t23 >> 2, 0x6420);
}

__device__ __forceinline__ uint32_t pair_sum16(uint32_t v)
{
    return (v & 0xFFFFu) + (v >> 16);
}

// Four consecutive DCT-input samples x = 4xg..4xg+3 of row y of one unit, as
// byte planes lo (and hi for 10-bit).  hv/wv: valid rows/columns of the unit in
// source samples (edge replication by clamping); xpart: wv < block width.
// HALF (10-bit H10 path): lo = f16x2 {x0, x1}, hi = f16x2 {x2, x3}, each sample v <= 1023
// as the f16 bit pattern 0x6400 | v, i.e. the value 1024 + v (exact; the 1024 offset is
// removed in dct16h / dct8pairh).
template <class F, int PL, bool HALF = false>
__device__ __forceinline__ void load4(uint32_t box, int ub, int y, int xg, int hv, int wv, bool xpart,
                                      uint32_t &lo, uint32_t &hi)
{
    constexpr int IB = PL == 0 ? F::IB_Y : F::IB_C;
    constexpr int RB = PL == 0 ? F::RB_Y : F::RB_C;
    constexpr int ES = F::ES;
    const int ub0 = ub * RB;
    if (!xpart) {
        if (!F::LP) {
            const int row = min(y, hv - 1);
            if (ES == 1) {
                lo = lds32(box + swz<IB>(row * IB + ub0 + 4 * xg));
                hi = 0;
            } else {
                uint2 v = lds64(box + swz<IB>(row * IB + ub0 + 8 * xg));
                v.x = __vminu2(v.x, 0x03FF03FFu);
                v.y = __vminu2(v.y, 0x03FF03FFu);
                if (HALF) {
                    lo = v.x | 0x64006400u;
                    hi = v.y | 0x64006400u;
                } else {
                    lo = __byte_perm(v.x, v.y, 0x6420);
                    hi = __byte_perm(v.x, v.y, 0x7531);
                }
            }
        } else {
            const int r0 = min(2 * y, hv - 1), r1 = min(2 * y + 1, hv - 1);
            if (ES == 1) {
                const uint2 a = lds64(box + swz<IB>(r0 * IB + ub0 + 8 * xg));
                const uint2 b = lds64(box + swz<IB>(r1 * IB + ub0 + 8 * xg));
                lo = ds8(a, b);
                hi = 0;
            } else {
                uint4 a = lds128(box + swz<IB>(r0 * IB + ub0 + 16 * xg));
                uint4 b = lds128(box + swz<IB>(r1 * IB + ub0 + 16 * xg));
                const uint32_t C10 = 0x03FF03FFu;
                const uint32_t d0 = (pair_sum16(__vminu2(a.x, C10)) + pair_sum16(__vminu2(b.x, C10)) + 2) >> 2;
                const uint32_t d1 = (pair_sum16(__vminu2(a.y, C10)) + pair_sum16(__vminu2(b.y, C10)) + 2) >> 2;
                const uint32_t d2 = (pair_sum16(__vminu2(a.z, C10)) + pair_sum16(__vminu2(b.z, C10)) + 2) >> 2;
                const uint32_t d3 = (pair_sum16(__vminu2(a.w, C10)) + pair_sum16(__vminu2(b.w, C10)) + 2) >> 2;
                const uint32_t p01 = d0 | (d1 << 16), p23 = d2 | (d3 << 16);
                if (HALF) {
                    lo = p01 | 0x64006400u;
                    hi = p23 | 0x64006400u;
                } else {
                    lo = __byte_perm(p01, p23, 0x6420);
                    hi = __byte_perm(p01, p23, 0x7531);
                }
            }
        }
    } else {  // partial last block column: per-sample clamped reads
        uint32_t l = 0, h = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int x = 4 * xg + k;
            int v;
            if (!F::LP) {
                v = box_sample<ES, IB>(box, ub0, min(y, hv - 1), min(x, wv - 1));
            } else {
                const int r0 = min(2 * y, hv - 1), r1 = min(2 * y + 1, hv - 1);
                const int x0 = min(2 * x, wv - 1), x1 = min(2 * x + 1, wv - 1);
                v = (box_sample<ES, IB>(box, ub0, r0, x0) + box_sample<ES, IB>(box, ub0, r0, x1) +
                     box_sample<ES, IB>(box, ub0, r1, x0) + box_sample<ES, IB>(box, ub0, r1, x1) + 2) >> 2;
            }
            if (HALF) {
                if (k < 2)
                    l |= (uint32_t)(v | 0x6400) << (16 * k);
                else
                    h |= (uint32_t)(v | 0x6400) << (16 * (k - 2));
            } else {
                l |= (uint32_t)(v & 255) << (8 * k);
                h |= (uint32_t)(v >> 8) << (8 * k);
            }
        }
        lo = l;
        hi = h;
    }
}

// ------------------------------------------------------------------ per-lane constant fragments
struct LaneConst {
    // n = 16 (m16n8k16): pass-1 A = T16, pass-2 A = T16[:, pi16]
    uint32_t t16a0, t16a1, p16a0, p16a1;
    // paired n = 8: pass-1 A = blockdiag(T8, T8), pass-2 A = blockdiag permuted
    uint32_t t8a0, t8a1, p8a0, p8a1;
    // n = 32 (m16n8k32), per m-tile
    uint32_t t32[2][4], p32[2][4];
    // 2x2 low-pass as an MMA: B = 0/1 pair-sum matrix, k = 4t+i (+16) -> source column,
    // n = g -> output column; luma rl = [2t + (i>>1) == g], chroma rc = same over 16 columns
    uint32_t rl, rc;
    // 10-bit f16 pass 1 (H10): A fragments (f16x2) of T16 and blockdiag(T8, T8) with the
    // contraction slots permuted to the load4<HALF> sample order, and the lane-0 DC
    // corrections of the pass-2 accumulators (dct16h, dct8pairh)
    uint32_t h16[4], h8[4];
    int32_t dcfix16, dcfix8e, dcfix8o;
    // n = 4 chroma of the n = 8 families (dct4oct): pass-1 A = blockdiag(T4 x 4) over
    // (unit, x), pass-2 A = blockdiag over (unit half, plane) with the pi4 slot order
    uint32_t t4a0, t4a1, p4a0, p4a1;
    // 8-bit two-plane f16 pass 2 (VCA_F16P2, dct16 / dct8pair): f16 A fragments of T16 and of
    // T8 in the standard contraction order, the pass-1 offset of this lane's row g (0 for the
    // DC row, 2^17 otherwise) and the hi-plane accumulator inits carrying the offset's
    // correction of the C_0k (k != 0) row
    // (the accumulator quads are loaded opaquely, so they stay resident instead of being
    // rebuilt with 4 moves per MMA; the corrections sit in the combine constants)
    uint32_t g16[4], g8;
    int32_t zq[4];      // pass-1 init {off_g, off_g, 2^17, 2^17}, off_g = 0 for g = 0, else 2^17
    float mq[4];        // pass-2 init 0.75 (bits 0x3F400000)
    int32_t kL0, kL1, kC0, kC1;  // combine constants -0x7F400000 - r_0 off_k (luma / chroma)
    int32_t mL0, mL1, mC0, mC1, mK;  // VCA_MIXP2 lo-plane accumulator inits -256 * 0x3F400000 - r_0 off_k
};

__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d)
{
    return (uint32_t)(a & 255) | ((uint32_t)(b & 255) << 8) | ((uint32_t)(c & 255) << 16) | ((uint32_t)(d & 255) << 24);
}

// pi16(k): slot k = 4t' + i' of pass 2 carries y = 8(i'>>1) + 2t' + (i'&1)
__device__ __forceinline__ int pi16(int k) { return 8 * ((k & 3) >> 1) + 2 * (k >> 2) + (k & 1); }
// pi32(k): k = 16h + 4t' + i' -> 16h + 8(i'>>1) + 2t' + (i'&1)
__device__ __forceinline__ int pi32(int k) { return 16 * (k >> 4) + pi16(k & 15); }

__device__ void build_lane_const(LaneConst &L, const int8_t *__restrict__ T_all, int g, int t, int NY)
{
    if (NY == 8 || NY == 16 || NY == 32) {
        const int8_t *T16 = T_all + table_offset(16);
        const int8_t *T8 = T_all + table_offset(8);
        auto T16a = [&](int i, int x) { return (int)__ldg(T16 + i * 16 + x); };
        auto T8a = [&](int i, int x) { return (int)__ldg(T8 + i * 8 + x); };
        L.t16a0 = pack4(T16a(g, 4 * t), T16a(g, 4 * t + 1), T16a(g, 4 * t + 2), T16a(g, 4 * t + 3));
        L.t16a1 = pack4(T16a(g + 8, 4 * t), T16a(g + 8, 4 * t + 1), T16a(g + 8, 4 * t + 2), T16a(g + 8, 4 * t + 3));
        L.p16a0 = pack4(T16a(g, pi16(4 * t)), T16a(g, pi16(4 * t + 1)), T16a(g, pi16(4 * t + 2)),
                        T16a(g, pi16(4 * t + 3)));
        L.p16a1 = pack4(T16a(g + 8, pi16(4 * t)), T16a(g + 8, pi16(4 * t + 1)), T16a(g + 8, pi16(4 * t + 2)),
                        T16a(g + 8, pi16(4 * t + 3)));
        // blockdiag(T8, T8): rows 0-7 (U) act on k 0-7, rows 8-15 (V) on k 8-15
        const int xb = 4 * (t & 1);
        const uint32_t row = pack4(T8a(g, xb), T8a(g, xb + 1), T8a(g, xb + 2), T8a(g, xb + 3));
        L.t8a0 = t < 2 ? row : 0u;
        L.t8a1 = t < 2 ? 0u : row;
        // pass 2: slot 4t+i carries (block (i>>1): 0 = U, 1 = V, y = 2t + (i&1))
        int u[4], v[4];
        for (int i = 0; i < 4; ++i) {
            const int y = 2 * t + (i & 1);
            const bool isV = (i >> 1) != 0;
            u[i] = isV ? 0 : T8a(g, y);
            v[i] = isV ? T8a(g, y) : 0;
        }
        L.p8a0 = pack4(u[0], u[1], u[2], u[3]);
        L.p8a1 = pack4(v[0], v[1], v[2], v[3]);
        auto h2 = [](int a, int b) {
            return (uint32_t)__half_as_ushort(__int2half_rn(a)) | ((uint32_t)__half_as_ushort(__int2half_rn(b)) << 16);
        };
        L.g16[0] = h2(T16a(g, 2 * t), T16a(g, 2 * t + 1));
        L.g16[1] = h2(T16a(g + 8, 2 * t), T16a(g + 8, 2 * t + 1));
        L.g16[2] = h2(T16a(g, 2 * t + 8), T16a(g, 2 * t + 9));
        L.g16[3] = h2(T16a(g + 8, 2 * t + 8), T16a(g + 8, 2 * t + 9));
        L.g8 = h2(T8a(g, 2 * t), T8a(g, 2 * t + 1));
        const int zoff = g == 0 ? 0 : (1 << 17);
        // opaque zero: T16[0][0] - 64 (the compiler cannot fold a loaded value)
        // (four distinct loads, so the four copies stay distinct registers of one quad)
        const int z0 = T16a(0, 0) - 64;
        L.zq[0] = zoff + z0;
        L.zq[1] = zoff + T16a(0, 1) - 64;
        L.zq[2] = (1 << 17) + T16a(0, 2) - 64;
        L.zq[3] = (1 << 17) + T16a(0, 3) - 64;
#pragma unroll
        for (int i = 0; i < 4; ++i) L.mq[i] = __int_as_float(0x3F400000 + T16a(0, 4 + i) - 64);
        // correction r_0 off_k of C_0k (r_0 = 64 n: 2^27 for n = 16, 2^26 for n = 8)
        const int32_t K = (int32_t)(0u - 0x7F400000u) + z0;
        L.kL0 = (g == 0 && t != 0) ? K - (1 << 27) : K;
        L.kL1 = g == 0 ? K - (1 << 27) : K;
        L.kC0 = (g == 0 && t != 0) ? K - (1 << 26) : K;
        L.kC1 = g == 0 ? K - (1 << 26) : K;
        // mixed pass 2 (VCA_MIXP2): C = E_lo + 256 bits(E_hi) - 256 * 0x3F400000 - r_0 off_k, the constant
        // in the lo-plane IMMA's accumulator (256 * 0x3F400000 = 0x40000000 mod 2^32)
        const int32_t KB = (int32_t)(0u - 0x40000000u) + z0;
        L.mL0 = (g == 0 && t != 0) ? KB - (1 << 27) : KB;
        L.mL1 = g == 0 ? KB - (1 << 27) : KB;
        L.mC0 = (g == 0 && t != 0) ? KB - (1 << 26) : KB;
        L.mC1 = g == 0 ? KB - (1 << 26) : KB;
        L.mK = KB;
    }
    {
        uint32_t r = 0;
        for (int i = 0; i < 4; ++i)
            if (2 * t + (i >> 1) == g) r |= 1u << (8 * i);
        L.rl = r;
        L.rc = r;
    }
    if (NY == 8) {
        // dct4oct.  Pass 1: row m = (b = m >> 2, j = m & 3), slot k = 4t + i = (b' = t, x = i):
        // A = T4[j][x] if b == b'.  Pass 2: row m' = (beta' = m' >> 3, c' = (m' >> 2) & 1, i' = m' & 3),
        // slot k' = 4t + i = (beta = i >> 1, c = t >> 1, y = 2 (t & 1) + (i & 1)):
        // A' = T4[i'][y] if beta' == beta and c' == c.  Lane rows are g (a0) and g + 8 (a1).
        const int8_t *T4 = T_all + table_offset(4);
        auto T4a = [&](int i, int x) { return (int)__ldg(T4 + i * 4 + x); };
        int v0[4], v1[4], w0[4], w1[4];
        for (int i = 0; i < 4; ++i) {
            v0[i] = t == (g >> 2) ? T4a(g & 3, i) : 0;
            v1[i] = t == 2 + (g >> 2) ? T4a(g & 3, i) : 0;
            const int y = 2 * (t & 1) + (i & 1);
            const bool cmatch = (t >> 1) == (g >> 2);
            w0[i] = (cmatch && (i >> 1) == 0) ? T4a(g & 3, y) : 0;
            w1[i] = (cmatch && (i >> 1) == 1) ? T4a(g & 3, y) : 0;
        }
        L.t4a0 = pack4(v0[0], v0[1], v0[2], v0[3]);
        L.t4a1 = pack4(v1[0], v1[1], v1[2], v1[3]);
        L.p4a0 = pack4(w0[0], w0[1], w0[2], w0[3]);
        L.p4a1 = pack4(w1[0], w1[1], w1[2], w1[3]);
    }
    if (NY == 16) {
        // f16 A fragment (m16n8k16, row-major): reg 0 = A[g][2t, 2t+1], 1 = A[g+8][2t, 2t+1],
        // 2 = A[g][2t+8, 2t+9], 3 = A[g+8][2t+8, 2t+9]; contraction slot (lane t, s) holds the
        // sample load4<HALF> put there: s = 0, 1 -> x = 4t + s (reg lo), s = 2, 3 -> x = 4t + s (reg hi)
        const int8_t *T16 = T_all + table_offset(16);
        const int8_t *T8 = T_all + table_offset(8);
        auto h2 = [](int a, int b) {
            return (uint32_t)__half_as_ushort(__int2half_rn(a)) | ((uint32_t)__half_as_ushort(__int2half_rn(b)) << 16);
        };
        auto T16a = [&](int i, int x) { return (int)__ldg(T16 + i * 16 + x); };
        auto T8a = [&](int i, int x) { return (int)__ldg(T8 + i * 8 + x); };
        L.h16[0] = h2(T16a(g, 4 * t), T16a(g, 4 * t + 1));
        L.h16[1] = h2(T16a(g + 8, 4 * t), T16a(g + 8, 4 * t + 1));
        L.h16[2] = h2(T16a(g, 4 * t + 2), T16a(g, 4 * t + 3));
        L.h16[3] = h2(T16a(g + 8, 4 * t + 2), T16a(g + 8, 4 * t + 3));
        // chroma pair: lanes t < 2 load U columns 4(t&1).., lanes t >= 2 V; rows g: U freq g,
        // rows g + 8: V freq g
        const bool isU = t < 2;
        const int xb = 4 * (t & 1);
        L.h8[0] = isU ? h2(T8a(g, xb), T8a(g, xb + 1)) : 0u;
        L.h8[1] = isU ? 0u : h2(T8a(g, xb), T8a(g, xb + 1));
        L.h8[2] = isU ? h2(T8a(g, xb + 2), T8a(g, xb + 3)) : 0u;
        L.h8[3] = isU ? 0u : h2(T8a(g, xb + 2), T8a(g, xb + 3));
        // pass-2 accumulator corrections, mod 2^32 (dct16h / dct8pairh): the pixel offset 1024
        // adds 1024 (64n)^2 to C_00 (2^30 for n = 16, 2^28 for n = 8); the plane-2 offset 64
        // adds 2^16 * 64 * 64n to every C_0j (2^32 == 0 for n = 16, 2^31 for n = 8).  Lanes g = 0
        // hold row i = 0; lane 0 slots e = 0 (and e = 2 for the V block) hold C_00.
        L.dcfix16 = (g == 0 && t == 0) ? (int32_t)(0u - (1u << 30)) : 0;
        L.dcfix8e = g == 0 ? (int32_t)((1u << 31) - (t == 0 ? (1u << 28) : 0u)) : 0;
        L.dcfix8o = g == 0 ? (int32_t)(1u << 31) : 0;
    }
    if (NY == 32) {
        const int8_t *T32 = T_all + table_offset(32);
        auto T32a = [&](int i, int x) { return (int)__ldg(T32 + i * 32 + x); };
        for (int mt = 0; mt < 2; ++mt) {
            const int r0 = 16 * mt + g, r1 = r0 + 8;
            L.t32[mt][0] = pack4(T32a(r0, 4 * t), T32a(r0, 4 * t + 1), T32a(r0, 4 * t + 2), T32a(r0, 4 * t + 3));
            L.t32[mt][1] = pack4(T32a(r1, 4 * t), T32a(r1, 4 * t + 1), T32a(r1, 4 * t + 2), T32a(r1, 4 * t + 3));
            L.t32[mt][2] = pack4(T32a(r0, 16 + 4 * t), T32a(r0, 17 + 4 * t), T32a(r0, 18 + 4 * t), T32a(r0, 19 + 4 * t));
            L.t32[mt][3] = pack4(T32a(r1, 16 + 4 * t), T32a(r1, 17 + 4 * t), T32a(r1, 18 + 4 * t), T32a(r1, 19 + 4 * t));
            L.p32[mt][0] = pack4(T32a(r0, pi32(4 * t)), T32a(r0, pi32(4 * t + 1)), T32a(r0, pi32(4 * t + 2)),
                                 T32a(r0, pi32(4 * t + 3)));
            L.p32[mt][1] = pack4(T32a(r1, pi32(4 * t)), T32a(r1, pi32(4 * t + 1)), T32a(r1, pi32(4 * t + 2)),
                                 T32a(r1, pi32(4 * t + 3)));
            L.p32[mt][2] = pack4(T32a(r0, pi32(16 + 4 * t)), T32a(r0, pi32(17 + 4 * t)), T32a(r0, pi32(18 + 4 * t)),
                                 T32a(r0, pi32(19 + 4 * t)));
            L.p32[mt][3] = pack4(T32a(r1, pi32(16 + 4 * t)), T32a(r1, pi32(17 + 4 * t)), T32a(r1, pi32(18 + 4 * t)),
                                 T32a(r1, pi32(19 + 4 * t)));
        }
    }
}

// ------------------------------------------------------------------ DCT building blocks
// n = 16: B fragments (lo/hi) for pass-1 n-tiles q = 0, 1 (y = 8q + g, x = 4t..4t+3)
// -> C[p][e]: i = g + 8(e>>1), j = 8p + 2t + (e&1).
// PERM1: the B fragments hold x in the pi16 slot order (tensor-core low-pass output),
// so pass 1 uses the column-permuted basis T16[:, pi16] -- the same constant as pass 2.
// 8-bit pass 2 as two f16 planes (VCA_F16P2, off: exact and parity-green, but slower).
// Pass 1 adds off_k = 2^17 to every row k != 0 through its accumulator (the DC row is >= 0
// already; the paired-n = 8 V rows take it at k = 0 too): with row sums r_k = 0 for k > 0
// and sum_x |T_kx| <= 64 n, every Z' = Z + off_k lies in [0, 2^18) for n <= 16 and 8-bit x,
// so byte 0 (lo) and bytes 1-2 (hi < 1024) of Z' are exact f16 subnormals lo * 2^-24,
// hi * 2^-24, each picked into the pass-2 B fragment by one PRMT (byte 3 of Z' is 0).  The
// pass-1 C fragment is the f16 B fragment as is (rows -> n, columns y = 2t, 2t+1 (+8) -> k),
// so A = T in the standard order.  With the f32 accumulator at 0.75 every partial sum is a
// multiple of 2^-24 in (0, 1): exact, and the result's bits are 0x3F400000 + S.  Then
// C = S_lo + 2^8 S_hi - r_i off_k = bits_lo + 2^8 bits_hi - 0x7F400000 - r_i off_k (mod 2^32).
// 4 PRMT + 2 HMMA instead of 7 PRMT + 3 IMMA per 4 values, yet config 3 -5 %, config 2 -14 %
// (profiles/r01d/ab_f16_pass2_reverted.log): the f32 HMMA costs more than the IMMAs it
// replaces and the resident accumulator quads add register pressure.
#ifndef VCA_F16P2
#define VCA_F16P2 0
#endif

// Mixed 8-bit pass 2 (VCA_MIXP2, default): with the same pass-1 offsets as VCA_F16P2 (every Z' in
// [0, 2^18)), the low byte of Z' goes through ONE s8 x u8 IMMA (the byte-plane path's plane 0)
// and Z' >> 8 (< 1024) through ONE f16 HMMA as exact subnormals (f32 accumulator at 0.75, so the
// result's bits are 0x3F400000 + S_hi, |S_hi| < 2^22); then C = E_lo + 256 bits(E_hi) with all
// constants in the IMMA's accumulator init: 5 PRMT + 1 IMMA + 1 HMMA + 1 IMAD per 4 values instead
// of 7 PRMT + 3 IMMA + 2 IMAD.  Exact (integer sums below 2^24 in f32), bit-identical results --
// but one f32 HMMA costs the tensor pipe more than the two IMMAs it replaces: config 3 -4 %,
// config 2 -6.6 % (profiles/r02/ab_mixed_pass2_reverted.log); off.
#ifndef VCA_MIXP2
#define VCA_MIXP2 0
#endif

template <int ES, bool PERM1 = false>
__device__ __forceinline__ void dct16(const LaneConst &L, const uint32_t (&blo)[2], const uint32_t (&bhi)[2],
                                      int32_t (&C)[2][4])
{
    int32_t D1[2][4];
    if (ES == 1 && VCA_MIXP2 && !VCA_F16P2) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
            mma16_su_c(D1[q], PERM1 ? L.p16a0 : L.t16a0, PERM1 ? L.p16a1 : L.t16a1, blo[q], L.zq[0], L.zq[1], L.zq[2],
                       L.zq[3]);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const uint32_t v0 = D1[0][2 * p], v1 = D1[0][2 * p + 1], v2 = D1[1][2 * p], v3 = D1[1][2 * p + 1];
            const uint32_t lo = __byte_perm(__byte_perm(v0, v1, 0x5140), __byte_perm(v2, v3, 0x5140), 0x5410);
            const uint32_t h0 = __byte_perm(v0, v1, 0x6521), h1 = __byte_perm(v2, v3, 0x6521);
            int32_t E0[4];
            mma16_su_c(E0, L.p16a0, L.p16a1, lo, p == 0 ? L.mL0 : L.mL1, L.mL1, L.mK, L.mK);
            float Eh[4];
            mma16_hc(Eh, L.g16[0], L.g16[1], L.g16[2], L.g16[3], h0, h1, L.mq[0], L.mq[1], L.mq[2], L.mq[3]);
#pragma unroll
            for (int e = 0; e < 4; ++e) C[p][e] = (int32_t)((uint32_t)E0[e] + __float_as_uint(Eh[e]) * 256u);
        }
        return;
    }
    if (ES == 1 && VCA_F16P2) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
            mma16_su_c(D1[q], PERM1 ? L.p16a0 : L.t16a0, PERM1 ? L.p16a1 : L.t16a1, blo[q], L.zq[0], L.zq[1], L.zq[2],
                       L.zq[3]);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const uint32_t lo0 = __byte_perm(D1[0][2 * p], D1[0][2 * p + 1], 0x7430);
            const uint32_t lo1 = __byte_perm(D1[1][2 * p], D1[1][2 * p + 1], 0x7430);
            const uint32_t hi0 = __byte_perm(D1[0][2 * p], D1[0][2 * p + 1], 0x6521);
            const uint32_t hi1 = __byte_perm(D1[1][2 * p], D1[1][2 * p + 1], 0x6521);
            float El[4], Eh[4];
            mma16_hc(El, L.g16[0], L.g16[1], L.g16[2], L.g16[3], lo0, lo1, L.mq[0], L.mq[1], L.mq[2], L.mq[3]);
            mma16_hc(Eh, L.g16[0], L.g16[1], L.g16[2], L.g16[3], hi0, hi1, L.mq[0], L.mq[1], L.mq[2], L.mq[3]);
            const int32_t K0 = p == 0 ? L.kL0 : L.kL1, K1 = L.kL1, K2 = (int32_t)(0u - 0x7F400000u);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                C[p][e] = (int32_t)(__float_as_uint(Eh[e]) * 256u + __float_as_uint(El[e]) +
                                    (uint32_t)(e == 0 ? K0 : e == 1 ? K1 : K2));
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (PERM1)
            mma16_su(D1[q], L.p16a0, L.p16a1, blo[q]);
        else
            mma16_su(D1[q], L.t16a0, L.t16a1, blo[q]);
        if (ES == 2) {
            int32_t Dh[4];
            mma16_su(Dh, L.t16a0, L.t16a1, bhi[q]);
#pragma unroll
            for (int e = 0; e < 4; ++e) D1[q][e] = (int32_t)((uint32_t)D1[q][e] + ((uint32_t)Dh[e] << 8));
        }
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        uint32_t b0, b1, b2;
        byte_planes(D1[0][2 * p], D1[0][2 * p + 1], D1[1][2 * p], D1[1][2 * p + 1], b0, b1, b2);
        int32_t E0[4], E1[4], E2[4];
        mma16_su(E0, L.p16a0, L.p16a1, b0);
        mma16_su(E1, L.p16a0, L.p16a1, b1);
        mma16_ss(E2, L.p16a0, L.p16a1, b2);
#pragma unroll
        for (int e = 0; e < 4; ++e) C[p][e] = combine3(E0[e], E1[e], E2[e]);
    }
}

// paired n = 8 (U rows 0-7 | V rows 8-15): one B fragment (thread t < 2: U x = 4t..,
// t >= 2: V x = 4(t-2)..; y = g) -> C[e]: e=0,1: U (i = g, j = 2t+e); e=2,3: V (i = g, j = 2t+e-2)
template <int ES, bool PERM1 = false>
__device__ __forceinline__ void dct8pair(const LaneConst &L, uint32_t blo, uint32_t bhi, int32_t (&C)[4])
{
    int32_t D1[4];
    if (ES == 1 && VCA_MIXP2 && !VCA_F16P2) {
        // as dct16's mixed pass 2; V rows take the 2^17 offset also at k = 0 (the luma pass-1 quad)
        mma16_su_c(D1, PERM1 ? L.p8a0 : L.t8a0, PERM1 ? L.p8a1 : L.t8a1, blo, L.zq[0], L.zq[1], L.zq[2], L.zq[3]);
        const uint32_t lo =
            __byte_perm(__byte_perm(D1[0], D1[1], 0x5140), __byte_perm(D1[2], D1[3], 0x5140), 0x5410);
        const uint32_t h0 = __byte_perm(D1[0], D1[1], 0x6521), h1 = __byte_perm(D1[2], D1[3], 0x6521);
        int32_t E0[4];
        mma16_su_c(E0, L.p8a0, L.p8a1, lo, L.mC0, L.mC1, L.mC1, L.mC1);
        float Eh[4];
        mma16_hc(Eh, L.g8, 0u, 0u, L.g8, h0, h1, L.mq[0], L.mq[1], L.mq[2], L.mq[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e) C[e] = (int32_t)((uint32_t)E0[e] + __float_as_uint(Eh[e]) * 256u);
        return;
    }
    if (ES == 1 && VCA_F16P2) {
        // V rows take the 2^17 offset also at k = 0 (Z_0 + 2^17 < 2^18 for n = 8), so the
        // pass-1 quad is the luma one; corrections: U C_0k (k != 0), V C_0k (all k)
        mma16_su_c(D1, PERM1 ? L.p8a0 : L.t8a0, PERM1 ? L.p8a1 : L.t8a1, blo, L.zq[0], L.zq[1], L.zq[2], L.zq[3]);
        const uint32_t lo0 = __byte_perm(D1[0], D1[1], 0x7430), lo1 = __byte_perm(D1[2], D1[3], 0x7430);
        const uint32_t hi0 = __byte_perm(D1[0], D1[1], 0x6521), hi1 = __byte_perm(D1[2], D1[3], 0x6521);
        float El[4], Eh[4];
        mma16_hc(El, L.g8, 0u, 0u, L.g8, lo0, lo1, L.mq[0], L.mq[1], L.mq[2], L.mq[3]);
        mma16_hc(Eh, L.g8, 0u, 0u, L.g8, hi0, hi1, L.mq[0], L.mq[1], L.mq[2], L.mq[3]);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            C[e] = (int32_t)(__float_as_uint(Eh[e]) * 256u + __float_as_uint(El[e]) + (uint32_t)(e == 0 ? L.kC0 : L.kC1));
        return;
    }
    if (PERM1)
        mma16_su(D1, L.p8a0, L.p8a1, blo);  // slot 4t+i = (U|V by i>>1, x = 2t + (i&1))
    else
        mma16_su(D1, L.t8a0, L.t8a1, blo);
    if (ES == 2) {
        int32_t Dh[4];
        mma16_su(Dh, L.t8a0, L.t8a1, bhi);
#pragma unroll
        for (int e = 0; e < 4; ++e) D1[e] = (int32_t)((uint32_t)D1[e] + ((uint32_t)Dh[e] << 8));
    }
    uint32_t b0, b1, b2;
    byte_planes(D1[0], D1[1], D1[2], D1[3], b0, b1, b2);
    int32_t E0[4], E1[4], E2[4];
    mma16_su(E0, L.p8a0, L.p8a1, b0);
    mma16_su(E1, L.p8a0, L.p8a1, b1);
    mma16_ss(E2, L.p8a0, L.p8a1, b2);
#pragma unroll
    for (int e = 0; e < 4; ++e) C[e] = combine3(E0[e], E1[e], E2[e]);
}



// 10-bit n = 16 (H10): pass 1 on the f16 tensor cores.  B = 1024 + x (load4<HALF>), A = T16
// (slot-permuted), C = 1.5 * 2^23: every product, partial sum and result is an integer of
// magnitude < 2^24 around 1.5 * 2^23, so the f32 accumulation is exact and the result's bit
// pattern is 0x4B400000 + Z' with Z' = Z + 2^20 [j = 0] (|Z'| < 2^22).  Its bytes 0, 1 are
// Z' mod 2^16 and byte 2 is (Z' >> 16) + 64 (u8), so pass 2 runs on those three planes as
// in dct16 (plane 2 unsigned) and the two offsets are removed mod 2^32 by the accumulator
// init of the plane-0 MMA (LaneConst::dcfix16).  Output layout identical to dct16.
__device__ __forceinline__ void dct16h(const LaneConst &L, const uint32_t (&blo)[2], const uint32_t (&bhi)[2],
                                       int32_t (&C)[2][4])
{
    int32_t D1[2][4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        float Df[4];
        mma16_h(Df, L.h16, blo[q], bhi[q], 12582912.0f);
#pragma unroll
        for (int e = 0; e < 4; ++e) D1[q][e] = __float_as_int(Df[e]);
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        uint32_t b0, b1, b2;
        byte_planes(D1[0][2 * p], D1[0][2 * p + 1], D1[1][2 * p], D1[1][2 * p + 1], b0, b1, b2);
        int32_t E0[4], E1[4], E2[4];
        if (p == 0)
            mma16_su_c(E0, L.p16a0, L.p16a1, b0, L.dcfix16, 0, 0, 0);
        else
            mma16_su(E0, L.p16a0, L.p16a1, b0);
        mma16_su(E1, L.p16a0, L.p16a1, b1);
        mma16_su(E2, L.p16a0, L.p16a1, b2);
#pragma unroll
        for (int e = 0; e < 4; ++e) C[p][e] = combine3(E0[e], E1[e], E2[e]);
    }
}

// 10-bit paired n = 8 (H10): as dct16h with A = blockdiag(T8, T8) (slot-permuted); the
// plane-2 offset adds 2^31 to every C_0j of both blocks and the pixel offset 2^28 to C_00
// (LaneConst::dcfix8e / dcfix8o).  Output layout identical to dct8pair.
__device__ __forceinline__ void dct8pairh(const LaneConst &L, uint32_t blo, uint32_t bhi, int32_t (&C)[4])
{
    float Df[4];
    mma16_h(Df, L.h8, blo, bhi, 12582912.0f);
    uint32_t b0, b1, b2;
    byte_planes(__float_as_int(Df[0]), __float_as_int(Df[1]), __float_as_int(Df[2]), __float_as_int(Df[3]), b0, b1,
                b2);
    int32_t E0[4], E1[4], E2[4];
    mma16_su_c(E0, L.p8a0, L.p8a1, b0, L.dcfix8e, L.dcfix8o, L.dcfix8e, L.dcfix8o);
    mma16_su(E1, L.p8a0, L.p8a1, b1);
    mma16_su(E2, L.p8a0, L.p8a1, b2);
#pragma unroll
    for (int e = 0; e < 4; ++e) C[e] = combine3(E0[e], E1[e], E2[e]);
}

// n = 4 chroma of 4 units x {U, V} = 8 blocks in one pass-1 and three pass-2 MMAs.  B fragment:
// lane (g, t) holds 4 samples x = 0..3 of row g & 3 of unit t's plane g >> 2 (U, V).  Output
// C[e]: plane g >> 2, i = g & 3, j = 2 (t & 1) + (e & 1), unit t >> 1 (e < 2) or 2 + (t >> 1).
template <int ES>
__device__ __forceinline__ void dct4oct(const LaneConst &L, uint32_t blo, uint32_t bhi, int32_t (&C)[4])
{
    int32_t D1[4];
    mma16_su(D1, L.t4a0, L.t4a1, blo);
    if (ES == 2) {
        int32_t Dh[4];
        mma16_su(Dh, L.t4a0, L.t4a1, bhi);
#pragma unroll
        for (int e = 0; e < 4; ++e) D1[e] = (int32_t)((uint32_t)D1[e] + ((uint32_t)Dh[e] << 8));
    }
    uint32_t b0, b1, b2;
    byte_planes(D1[0], D1[1], D1[2], D1[3], b0, b1, b2);
    int32_t E0[4], E1[4], E2[4];
    mma16_su(E0, L.p4a0, L.p4a1, b0);
    mma16_su(E1, L.p4a0, L.p4a1, b1);
    mma16_ss(E2, L.p4a0, L.p4a1, b2);
#pragma unroll
    for (int e = 0; e < 4; ++e) C[e] = combine3(E0[e], E1[e], E2[e]);
}

// Cross-lane sums of a warp's 6 per-item partials in one reduce-scatter (VCA_XRED8): 8 values
// (6 used) over 32 lanes; each xor round halves the values a lane carries (lanes keep one half
// and receive the partner's copy of it), so 4 + 2 + 1 + 1 + 1 = 9 double shuffles instead of
// 6 x 5.  Lane l ends with the total of value (l >> 2) & 7; the order is fixed.
#ifndef VCA_XRED8
#define VCA_XRED8 1
#endif
__device__ __forceinline__ double xred8(const double (&v)[8], int lane)
{
    const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
    double k[4], m[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double send = b4 ? v[i] : v[i + 4], keep = b4 ? v[i + 4] : v[i];
        k[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double send = b3 ? k[i] : k[i + 2], keep = b3 ? k[i + 2] : k[i];
        m[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const double send = b2 ? m[0] : m[1], keep = b2 ? m[1] : m[0];
    double n = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    n += __shfl_xor_sync(0xffffffffu, n, 2);
    n += __shfl_xor_sync(0xffffffffu, n, 1);
    return n;
}

#ifdef VCA_TIMES
// diagnostic build only (tools/group_times.py): per consumer group, globaltimer at its first
// wait and after its last item
__device__ unsigned long long vca_group_t[3][4096];  // start, end, SM id
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

// ------------------------------------------------------------------ kernel
struct FusedArgs {
    int n_frames;
    int width[3], height[3];
    int cols, rows;
    const double *W_all;
    const int8_t *T_all;
    Scratch s;
    DumpPtrs dump;
    // dynamic item scheduling (VCA_DYN): a context-owned ticket counter that is never reset;
    // this launch owns tickets [ticket_base, ticket_base + items + groups)
    unsigned long long *ticket;
    unsigned long long ticket_base;
    int y4, c4;  // the Y / chroma tensor maps are 4-D (one load per plane per strip)
};

// Work distribution over the consumer groups.  0: static round robin (item it goes to virtual
// CTA it mod (grid x groups)); 1: dynamic -- each group's producer takes the next item from a
// global ticket counter and passes its index to the consumers in a per-stage header word, so
// groups on faster SMs take more items and the launch ends when the work does, not when the
// slowest SM's fixed share does.  Results do not depend on the assignment (every item's sums
// are computed in a fixed order by whichever group takes it).
#ifndef VCA_DYN
#define VCA_DYN 0
#endif

// A ragged last strip (fewer whole units than a full strip: config 3's 120 block columns are
// 7.5 strips of 16) runs each warp's first two whole units as one 2-unit group instead of two
// single units (A/B: VCA_RAGGED2 0 / 1)
#ifndef VCA_RAGGED2
#define VCA_RAGGED2 1
#endif

template <class F>
struct UnitCtx {
    static constexpr int NWC = F::NC == 16 ? 8 : 2;
    LaneConst L;
    double wl16[8];     // luma n = 16 weights at this lane's 8 positions
    double wc[NWC];     // chroma weights at this lane's positions (NY = 8: the n = 8 luma pair's)
    double w4[2];       // NY = 8: n = 4 chroma weights at this lane's positions (dct4oct)
    uint32_t wtab;      // smem offset of this lane's luma n = 32 weights ([pair][lane] double2)
    uint32_t wsm;       // smem address of this lane's n = 16 / 8 weights ([e][lane])
    int g, t;
};

struct UnitOut {
    double hY;          // luma texture partial, summed over the 4 lanes of row group g
    double hu, hv;      // this lane's U / V texture partials
    int32_t dcY, dcU, dcV;  // C_00 (mod 2^32) in lane 0
};

// A2-A6 for NU units (each: Y block + U, V blocks) of one consumer warp:
// swizzled smem -> registers -> exact integer DCT on the tensor cores -> FP64
// weighted |C| partials.  The NU units are independent instruction streams the
// compiler interleaves (latency hiding within the warp).
#ifdef VCA_MMA_DS
constexpr bool kMmaDownsample = true;   // A/B: 2x2 low-pass sums as a 0/1 IMMA (exact, but its
#else                                   // latency sits on the critical path: -4 % vs the ALUs)
constexpr bool kMmaDownsample = false;
#endif

// Chroma needs only per-frame sums (A7), so a lane may add |C| per coefficient position into
// exact uint32 accumulators and apply the weight once per flush (every FC units; FC keeps
// the sums below 2^32: |C| <= (64 n)^2 (2^bd - 1) and FC * that < 2^32) -- no conversion or
// FP64 op per chroma coefficient, exact sums, only the flushes round.  A/B with the
// warp-specialised NU = 4 kernel (profiles/r01c/ab_intchroma.log): config 3 +1.9 % burst and
// +1.7 % under the 1000 W power cap, config 4 +10 %, config 2 +2 % -- on everywhere.
#ifndef VCA_INT_CHROMA
#define VCA_INT_CHROMA 2  // 0 never, 1 n = 16 chroma only, 2 always
#endif

template <class F>
struct ChromaAcc {
    static constexpr bool ON = VCA_INT_CHROMA == 2 || (VCA_INT_CHROMA == 1 && F::NC == 16);
    static constexpr int NP = F::NC == 16 ? 8 : 2;  // coefficient positions per lane per plane
    // units per flush: the largest power of two <= 64 with FC * (64 n)^2 (2^bd - 1) < 2^32
    // (n = 8 8-bit: 64; n = 8 10-bit and n = 16 8-bit: 16; n = 16 10-bit: 4); the n = 8 families
    // (several blocks per position per group) keep 16
    static constexpr uint64_t CMAX = (uint64_t)(64 * F::NC) * (64 * F::NC) * ((1u << F::BD) - 1u);
    static constexpr uint64_t FCMAX = 4294967295ull / CMAX;
    static constexpr int FC = F::NY == 8 ? 16 : FCMAX >= 64 ? 64 : FCMAX >= 32 ? 32 : FCMAX >= 16 ? 16 : FCMAX >= 8 ? 8 : 4;
    static_assert(F::NY == 8 || (uint64_t)FC * CMAX <= 4294967295ull, "chroma sums fit uint32");
    uint32_t u[NP], v[NP];
};


template <class F, bool XPART, bool DUMP, int NU>
__device__ __forceinline__ void process_units(const UnitCtx<F> &U, const FusedArgs &a, const uint32_t (&boxY)[NU],
                                              const uint32_t (&boxU)[NU], const int (&ubY)[NU],
                                              const int (&ubC)[NU], int hvY, int hvC, int wvY, int wvC,
                                              const int64_t (&k)[NU], UnitOut (&o)[NU], double &hu_acc,
                                              double &hv_acc, ChromaAcc<F> &ca)
{
    constexpr int NY = F::NY, NC = F::NC, ES = F::ES;
    const int g = U.g, t = U.t;
    const LaneConst &L = U.L;
    // weights from smem ([e][lane] doubles, conflict-free), loaded once per call
    double wl[8], wcc[2];
    if (NY == 16 && NC == 8) {
#pragma unroll
        for (int e = 0; e < 8; ++e) wl[e] = lds_f64(U.wsm + e * 256);
#pragma unroll
        for (int e = 0; e < 2; ++e) wcc[e] = lds_f64(U.wsm + (8 + e) * 256);
    } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) wl[e] = U.wl16[e];
#pragma unroll
        for (int e = 0; e < 2; ++e) wcc[e] = U.wc[e];
    }
    double hY[NU];
    int64_t ckY[NU], ckU[NU], ckV[NU];  // DUMP: per-lane AC checksum terms (tests)
#pragma unroll
    for (int n = 0; n < NU; ++n) ckY[n] = ckU[n] = ckV[n] = 0;
    // 8-bit low-pass on whole columns: the 2x2 sums run on the tensor cores (A3 as an
    // exact 0/1 contraction, rounding offset as the accumulator init)
    constexpr bool MMA_DS = F::LP && ES == 1 && !XPART && kMmaDownsample;
    if (NY == 16) {
        uint32_t blo[NU][2], bhi[NU][2];
        if (MMA_DS) {
            // S^T[y][x] = sum_{parity, col} px(2y + parity, col) [col/2 == x]: M = y (16),
            // N = x (2 n-tiles), K = 2 x 32 (row parity x source column)
            const int32_t two[4] = {2, 2, 2, 2};
#pragma unroll
            for (int n = 0; n < NU; ++n) {
                int32_t S[2][4];
                uint32_t A[2][4];
                const int ub0 = ubY[n] * F::RB_Y;
#pragma unroll
                for (int par = 0; par < 2; ++par) {
                    const int r0 = min(2 * g + par, hvY - 1), r1 = min(2 * (g + 8) + par, hvY - 1);
                    A[par][0] = lds32(boxY[n] + swz<F::IB_Y>(r0 * F::IB_Y + ub0 + 4 * t));
                    A[par][1] = lds32(boxY[n] + swz<F::IB_Y>(r1 * F::IB_Y + ub0 + 4 * t));
                    A[par][2] = lds32(boxY[n] + swz<F::IB_Y>(r0 * F::IB_Y + ub0 + 16 + 4 * t));
                    A[par][3] = lds32(boxY[n] + swz<F::IB_Y>(r1 * F::IB_Y + ub0 + 16 + 4 * t));
                }
                // n-tile 0 (x = g): source columns 0..15 only; n-tile 1 (x = 8 + g): 16..31
                mma32_uu_acc(S[0], A[0], L.rl, 0u, two);
                mma32_uu_acc(S[0], A[1], L.rl, 0u, S[0]);
                mma32_uu_acc(S[1], A[0], 0u, L.rl, two);
                mma32_uu_acc(S[1], A[1], 0u, L.rl, S[1]);
                // pass-1 B fragments in pi16 slot order: y = g from c0, c1; y = g + 8 from c2, c3
                blo[n][0] = pack_ds(S[0][0], S[0][1], S[1][0], S[1][1]);
                blo[n][1] = pack_ds(S[0][2], S[0][3], S[1][2], S[1][3]);
                bhi[n][0] = bhi[n][1] = 0;
            }
        } else {
#pragma unroll
            for (int n = 0; n < NU; ++n)
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    load4<F, 0, F::H10>(boxY[n], ubY[n], 8 * q + g, t, hvY, wvY, XPART, blo[n][q], bhi[n][q]);
        }
        int32_t C[NU][2][4];
#pragma unroll
        for (int n = 0; n < NU; ++n) {
            if (F::H10)
                dct16h(L, blo[n], bhi[n], C[n]);
            else
                dct16<ES, MMA_DS>(L, blo[n], bhi[n], C[n]);
        }
        if (DUMP || kMutate) {
#pragma unroll
            for (int n = 0; n < NU; ++n)
#pragma unroll
                for (int p = 0; p < 2; ++p)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int pos = (g + 8 * (e >> 1)) * 16 + 8 * p + 2 * t + (e & 1);
                        if (kMutate && pos) C[n][p][e] = mutate<DUMP>(C[n][p][e], 0, k[n], pos);
                        if (DUMP && pos) ckY[n] += (int64_t)C[n][p][e] * (pos + 1);
                    }
        }
#pragma unroll
        for (int n = 0; n < NU; ++n) {
            // |C| folds into the DFMA operand (fabs of an exact int32 -> double conversion)
            double h0 = 0.0, h1 = 0.0;  // two FMA chains, combined once (fixed order)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                h0 = fma(wl[e], fabs(i2d(C[n][0][e])), h0);
                h1 = fma(wl[4 + e], fabs(i2d(C[n][1][e])), h1);
            }
            hY[n] = h0 + h1;
            o[n].dcY = C[n][0][0];
            if (DUMP && a.dump.coeffs[0]) {
#pragma unroll
                for (int p = 0; p < 2; ++p)
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        a.dump.coeffs[0][k[n] * 256 + (g + 8 * (e >> 1)) * 16 + 8 * p + 2 * t + (e & 1)] = C[n][p][e];
            }
        }
    } else {
        // n = 32: pass 1 over 4 n-tiles (y = 8q + g), 2 m-tiles (j = 16mt + g (+8)); NU units
        // as independent instruction streams
        int32_t D1[NU][2][4][4];
#pragma unroll
        for (int n = 0; n < NU; ++n)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t l0, h0, l1, h1;
                load4<F, 0>(boxY[n], ubY[n], 8 * q + g, t, hvY, wvY, XPART, l0, h0);
                load4<F, 0>(boxY[n], ubY[n], 8 * q + g, 4 + t, hvY, wvY, XPART, l1, h1);
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    mma32_su(D1[n][mt][q], L.t32[mt], l0, l1);
                    if (ES == 2) {
                        int32_t Dh[4];
                        mma32_su(Dh, L.t32[mt], h0, h1);
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            D1[n][mt][q][e] = (int32_t)((uint32_t)D1[n][mt][q][e] + ((uint32_t)Dh[e] << 8));
                    }
                }
            }
        // four independent FMA chains per unit (one per fragment slot e), combined in a fixed order
        double hacc[NU][4];
#pragma unroll
        for (int n = 0; n < NU; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) hacc[n][e] = 0.0;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            const int ms = rr >> 1, hf = rr & 1;
#pragma unroll
            for (int n = 0; n < NU; ++n) {
                uint32_t b0a, b1a, b2a, b0b, b1b, b2b;
                byte_planes(D1[n][ms][0][2 * hf], D1[n][ms][0][2 * hf + 1], D1[n][ms][1][2 * hf],
                            D1[n][ms][1][2 * hf + 1], b0a, b1a, b2a);
                byte_planes(D1[n][ms][2][2 * hf], D1[n][ms][2][2 * hf + 1], D1[n][ms][3][2 * hf],
                            D1[n][ms][3][2 * hf + 1], b0b, b1b, b2b);
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    int32_t E0[4], E1[4], E2[4];
                    mma32_su(E0, L.p32[mt], b0a, b0b);
                    mma32_su(E1, L.p32[mt], b1a, b1b);
                    mma32_ss(E2, L.p32[mt], b2a, b2b);
                    const double2 w01 = lds<double2>(U.wtab + ((mt * 4 + rr) * 2 + 0) * 512);
                    const double2 w23 = lds<double2>(U.wtab + ((mt * 4 + rr) * 2 + 1) * 512);
                    const double wv[4] = {w01.x, w01.y, w23.x, w23.y};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        int32_t cc = combine3(E0[e], E1[e], E2[e]);
                        const int pos = (16 * mt + g + 8 * (e >> 1)) * 32 + 8 * rr + 2 * t + (e & 1);
                        if (kMutate && pos) cc = mutate<DUMP>(cc, 0, k[n], pos);
                        hacc[n][e] = fma(wv[e], fabs(i2d(cc)), hacc[n][e]);
                        if (mt == 0 && rr == 0 && e == 0) o[n].dcY = cc;
                        if (DUMP) {
                            if (pos) ckY[n] += (int64_t)cc * (pos + 1);
                            if (a.dump.coeffs[0]) a.dump.coeffs[0][k[n] * 1024 + pos] = cc;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int n = 0; n < NU; ++n) hY[n] = (hacc[n][0] + hacc[n][1]) + (hacc[n][2] + hacc[n][3]);
    }
#pragma unroll
    for (int n = 0; n < NU; ++n) {
        // reduce over the 4 lanes of a row group (lanes t == 0 hold the partial of rows g (+8, ...)),
        // or over lane pairs (HSLOTS == 16: lanes t = 0, 2 hold half a row group each)
        hY[n] += __shfl_xor_sync(0xffffffffu, hY[n], 1);
        if (F::HSLOTS == 8) hY[n] += __shfl_xor_sync(0xffffffffu, hY[n], 2);
        o[n].hY = hY[n];
    }

    // ---- chroma
    if (NC == 8) {
        uint32_t blo[NU], bhi[NU];
        if (MMA_DS) {
            // M = 16 (U rows y = m | V rows y = m - 8), N = x (8), K = row parity x 16 columns
            const int32_t two[4] = {2, 2, 2, 2};
#pragma unroll
            for (int n = 0; n < NU; ++n) {
                const int ub0 = ubC[n] * F::RB_C;
                const int r0 = min(2 * g, hvC - 1), r1 = min(2 * g + 1, hvC - 1);
                uint32_t A[4];
                A[0] = lds32(boxU[n] + swz<F::IB_C>(r0 * F::IB_C + ub0 + 4 * t));
                A[1] = lds32(boxU[n] + F::ST_C + swz<F::IB_C>(r0 * F::IB_C + ub0 + 4 * t));
                A[2] = lds32(boxU[n] + swz<F::IB_C>(r1 * F::IB_C + ub0 + 4 * t));
                A[3] = lds32(boxU[n] + F::ST_C + swz<F::IB_C>(r1 * F::IB_C + ub0 + 4 * t));
                int32_t S[4];
                mma32_uu_acc(S, A, L.rc, L.rc, two);
                // slots 4t+i: U x = 2t + i (i < 2), V x = 2t + i - 2 -> the p8 permutation
                blo[n] = pack_ds(S[0], S[1], S[2], S[3]);
                bhi[n] = 0;
            }
        } else {
#pragma unroll
            for (int n = 0; n < NU; ++n)
                load4<F, 1, F::H10>(t < 2 ? boxU[n] : boxU[n] + F::ST_C, ubC[n], g, t & 1, hvC, wvC, XPART, blo[n],
                                    bhi[n]);
        }
        int32_t C[NU][4];
#pragma unroll
        for (int n = 0; n < NU; ++n) {
            if (F::H10)
                dct8pairh(L, blo[n], bhi[n], C[n]);
            else
                dct8pair<ES, MMA_DS>(L, blo[n], bhi[n], C[n]);
        }
        if (DUMP || kMutate) {
#pragma unroll
            for (int n = 0; n < NU; ++n)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int pos = g * 8 + 2 * t + (e & 1);
                    if (kMutate && pos) C[n][e] = mutate<DUMP>(C[n][e], 1 + (e >> 1), k[n], pos);
                    if (DUMP && pos) (e < 2 ? ckU[n] : ckV[n]) += (int64_t)C[n][e] * (pos + 1);
                }
        }
#pragma unroll
        for (int n = 0; n < NU; ++n) {
            if (ChromaAcc<F>::ON) {
                ca.u[0] += (uint32_t)abs(C[n][0]);
                ca.u[1] += (uint32_t)abs(C[n][1]);
                ca.v[0] += (uint32_t)abs(C[n][2]);
                ca.v[1] += (uint32_t)abs(C[n][3]);
                if (DUMP) {
                    o[n].hu = fma(wcc[1], fabs(i2d(C[n][1])), wcc[0] * fabs(i2d(C[n][0])));
                    o[n].hv = fma(wcc[1], fabs(i2d(C[n][3])), wcc[0] * fabs(i2d(C[n][2])));
                }
            } else {
                o[n].hu = fma(wcc[1], fabs(i2d(C[n][1])), wcc[0] * fabs(i2d(C[n][0])));
                o[n].hv = fma(wcc[1], fabs(i2d(C[n][3])), wcc[0] * fabs(i2d(C[n][2])));
                hu_acc += o[n].hu;
                hv_acc += o[n].hv;
            }
            o[n].dcU = C[n][0];
            o[n].dcV = C[n][2];
            if (DUMP && a.dump.coeffs[1]) {
                a.dump.coeffs[1][k[n] * 64 + g * 8 + 2 * t] = C[n][0];
                a.dump.coeffs[1][k[n] * 64 + g * 8 + 2 * t + 1] = C[n][1];
            }
            if (DUMP && a.dump.coeffs[2]) {
                a.dump.coeffs[2][k[n] * 64 + g * 8 + 2 * t] = C[n][2];
                a.dump.coeffs[2][k[n] * 64 + g * 8 + 2 * t + 1] = C[n][3];
            }
        }
    } else {
#pragma unroll
        for (int n = 0; n < NU; ++n)
#pragma unroll
            for (int pl = 1; pl <= 2; ++pl) {
                const uint32_t box = pl == 1 ? boxU[n] : boxU[n] + F::ST_C;
                uint32_t blo[2], bhi[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) load4<F, 1>(box, ubC[n], 8 * q + g, t, hvC, wvC, XPART, blo[q], bhi[q]);
                int32_t C[2][4];
                dct16<ES>(L, blo, bhi, C);
                if (DUMP || kMutate) {
#pragma unroll
                    for (int p = 0; p < 2; ++p)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int pos = (g + 8 * (e >> 1)) * 16 + 8 * p + 2 * t + (e & 1);
                            if (kMutate && pos) C[p][e] = mutate<DUMP>(C[p][e], pl, k[n], pos);
                            if (DUMP && pos) (pl == 1 ? ckU[n] : ckV[n]) += (int64_t)C[p][e] * (pos + 1);
                        }
                }
                double hacc = 0.0;
                if (ChromaAcc<F>::ON) {
#pragma unroll
                    for (int p = 0; p < 2; ++p)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            if (pl == 1)
                                ca.u[p * 4 + e] += (uint32_t)abs(C[p][e]);
                            else
                                ca.v[p * 4 + e] += (uint32_t)abs(C[p][e]);
                        }
                }
                if (!ChromaAcc<F>::ON || DUMP) {
                    double h2[2] = {0.0, 0.0};  // two chains, fixed combination
#pragma unroll
                    for (int p = 0; p < 2; ++p)
#pragma unroll
                        for (int e = 0; e < 4; ++e) h2[p] = fma(U.wc[p * 4 + e], fabs(i2d(C[p][e])), h2[p]);
                    hacc = h2[0] + h2[1];
                }
                if (pl == 1) {
                    o[n].hu = hacc;
                    o[n].dcU = C[0][0];
                    if (!ChromaAcc<F>::ON) hu_acc += hacc;
                } else {
                    o[n].hv = hacc;
                    o[n].dcV = C[0][0];
                    if (!ChromaAcc<F>::ON) hv_acc += hacc;
                }
                if (DUMP && a.dump.coeffs[pl]) {
#pragma unroll
                    for (int p = 0; p < 2; ++p)
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            a.dump.coeffs[pl][k[n] * 256 + (g + 8 * (e >> 1)) * 16 + 8 * p + 2 * t + (e & 1)] = C[p][e];
                }
            }
    }
    if (DUMP) {
#pragma unroll
        for (int n = 0; n < NU; ++n) {
            double hy = hY[n], hu = o[n].hu, hv = o[n].hv;
#pragma unroll
            for (int s = F::HSLOTS == 8 ? 4 : 2; s < 32; s <<= 1) hy += __shfl_xor_sync(0xffffffffu, hy, s);
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
                hu += __shfl_xor_sync(0xffffffffu, hu, s);
                hv += __shfl_xor_sync(0xffffffffu, hv, s);
            }
            chk_add(a.dump.chk[0], k[n], ckY[n]);
            chk_add(a.dump.chk[1], k[n], ckU[n]);
            chk_add(a.dump.chk[2], k[n], ckV[n]);
            if (g == 0 && t == 0) {
                const uint32_t sx[3] = {(uint32_t)o[n].dcY >> 12, (uint32_t)o[n].dcU >> 12, (uint32_t)o[n].dcV >> 12};
                const double hh[3] = {hy, hu, hv};
                const int64_t kk = k[n];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    if (a.dump.sumx[q]) a.dump.sumx[q][kk] = sx[q];
                    if (a.dump.H[q]) a.dump.H[q][kk] = hh[q];
                    if (a.dump.L[q]) a.dump.L[q][kk] = sqrt((double)sx[q] * (q == 0 ? 1.0 / NY : 1.0 / NC));
                }
            }
        }
    }
}

// A2-A6 for the n = 8 families (w = 16 low-pass, w = 8 full): one consumer warp's 4 units of
// a strip.  Luma: two dct8pair calls (units 0|1 and 2|3 as the block-diagonal pair); chroma:
// one dct4oct for the 4 units x {U, V}.  Lane geometry (which unit a lane loads) is in LY*/LC*.
// XPART: per-lane valid widths (partial last block column; units past the frame read the
// zero-filled TMA box and are never stored).  Outputs: per-unit luma row-group partials hY
// (valid in lanes t == 0), the DC terms (luma in lane 0, chroma in the lanes holding them),
// exact chroma sums into ca.
template <class F, bool XPART, bool DUMP>
__device__ __forceinline__ void process_group8(const UnitCtx<F> &U, const FusedArgs &a, uint32_t base,
                                               const uint32_t (&LYoff)[2], const int (&LYub)[2], uint32_t LCoff,
                                               int LCub, int hvY, int hvC, const int (&wvY)[2], int wvC,
                                               const int64_t (&k)[4], double (&hY)[4], int32_t (&dcY)[4],
                                               int32_t (&dcC)[2], ChromaAcc<F> &ca)
{
    constexpr int ES = F::ES, W = F::W, WC = F::WC;
    const int g = U.g, t = U.t;
    const LaneConst &L = U.L;
    const double wc0 = U.wc[0], wc1 = U.wc[1];
    // ---- luma: pairs p = 0 (units 0, 1), 1 (units 2, 3); lane t < 2 loads the first unit
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        uint32_t lo, hi;
        load4<F, 0>(base + LYoff[p], LYub[p], g, t & 1, hvY, XPART ? wvY[p] : W, XPART && wvY[p] < W, lo, hi);
        int32_t C[4];
        dct8pair<ES>(L, lo, hi, C);
        if (DUMP || kMutate) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t kk = k[2 * p + (e >> 1)];
                const int pos = g * 8 + 2 * t + (e & 1);
                if (kMutate && pos && kk >= 0) C[e] = mutate<DUMP>(C[e], 0, kk, pos);
                if (DUMP && pos && kk >= 0) chk_add(a.dump.chk[0], kk, (int64_t)C[e] * (pos + 1));
            }
        }
        double h0 = fma(wc1, fabs(i2d(C[1])), wc0 * fabs(i2d(C[0])));
        double h1 = fma(wc1, fabs(i2d(C[3])), wc0 * fabs(i2d(C[2])));
        h0 += __shfl_xor_sync(0xffffffffu, h0, 1);
        h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
        h0 += __shfl_xor_sync(0xffffffffu, h0, 2);
        h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
        hY[2 * p] = h0;
        hY[2 * p + 1] = h1;
        dcY[2 * p] = C[0];
        dcY[2 * p + 1] = C[2];
        if (DUMP && a.dump.coeffs[0]) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t kk = k[2 * p + (e >> 1)];
                if (kk >= 0) a.dump.coeffs[0][kk * 64 + g * 8 + 2 * t + (e & 1)] = C[e];
            }
        }
    }
    // ---- chroma: 8 blocks of 4 x 4 (unit t, plane g >> 2, row g & 3)
    {
        uint32_t lo, hi;
        load4<F, 1>(base + LCoff, LCub, g & 3, 0, hvC, XPART ? wvC : WC, XPART && wvC < WC, lo, hi);
        int32_t C[4];
        dct4oct<ES>(L, lo, hi, C);
        if (DUMP || kMutate) {
            const int pl = 1 + (g >> 2);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t kk = k[e < 2 ? (t >> 1) : 2 + (t >> 1)];
                const int pos = (g & 3) * 4 + 2 * (t & 1) + (e & 1);
                if (kMutate && pos && kk >= 0) C[e] = mutate<DUMP>(C[e], pl, kk, pos);
                if (DUMP && pos && kk >= 0) chk_add(a.dump.chk[pl], kk, (int64_t)C[e] * (pos + 1));
            }
        }
        // lane's plane is fixed (g >> 2); slots e and e + 2 share a weight (different units)
        const uint32_t s0 = (uint32_t)abs(C[0]) + (uint32_t)abs(C[2]);
        const uint32_t s1 = (uint32_t)abs(C[1]) + (uint32_t)abs(C[3]);
        if (g < 4) {
            ca.u[0] += s0;
            ca.u[1] += s1;
        } else {
            ca.v[0] += s0;
            ca.v[1] += s1;
        }
        dcC[0] = C[0];
        dcC[1] = C[2];
        if (DUMP) {
            const int pl = 1 + (g >> 2);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t kk = k[e < 2 ? (t >> 1) : 2 + (t >> 1)];
                if (kk >= 0 && a.dump.coeffs[pl]) a.dump.coeffs[pl][kk * 16 + (g & 3) * 4 + 2 * (t & 1) + (e & 1)] = C[e];
            }
            // per-block chroma H: this lane's weighted terms, reduced over the warp per (unit, plane)
#pragma unroll
            for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    double v = 0.0;
                    if ((g >> 2) == q) {
                        if ((t >> 1) == n) v = fma(U.w4[1], fabs(i2d(C[1])), U.w4[0] * fabs(i2d(C[0])));
                        if (2 + (t >> 1) == n) v = fma(U.w4[1], fabs(i2d(C[3])), U.w4[0] * fabs(i2d(C[2])));
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if ((g | t) == 0 && k[n] >= 0 && a.dump.H[1 + q]) a.dump.H[1 + q][k[n]] = v;
                }
            // per-block chroma DC sums and L (lane (4q, 2 (n & 1)) holds unit n's plane-q DC)
            if ((g & 3) == 0 && (t & 1) == 0) {
                const int q = g >> 2;
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    const int n = m == 0 ? (t >> 1) : 2 + (t >> 1);
                    if (k[n] >= 0) {
                        const uint32_t sx = (uint32_t)dcC[m] >> 12;
                        if (a.dump.sumx[1 + q]) a.dump.sumx[1 + q][k[n]] = sx;
                        if (a.dump.L[1 + q]) a.dump.L[1 + q][k[n]] = sqrt((double)sx * (1.0 / F::NC));
                    }
                }
            }
        }
    }
    if (DUMP) {  // per-block luma H, DC sum, L
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            double v = hY[n];
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((g | t) == 0 && k[n] >= 0) {
                const uint32_t sx = (uint32_t)dcY[n] >> 12;
                if (a.dump.H[0]) a.dump.H[0][k[n]] = v;
                if (a.dump.sumx[0]) a.dump.sumx[0][k[n]] = sx;
                if (a.dump.L[0]) a.dump.L[0][k[n]] = sqrt((double)sx * (1.0 / F::NY));
            }
        }
    }
}

// CTA layouts.
//  * kGroups == 0: 160 threads = 1 producer warp + 4 consumer warps (A/B: a producer-less
//    ring refilled by the last releasing warp lost 16 %), MINB CTAs per SM.
//  * kGroups == G > 0: warp-specialised with register reallocation, 1 CTA per SM:
//    warpgroup 0 = producers (warp g < G feeds group g; setmaxnreg.dec to VCA_PREG),
//    warpgroups 1..G = consumer groups of 4 warps (setmaxnreg.inc to VCA_CREG), each group
//    with its own ring, walking its own item sequence exactly like one legacy CTA.
// Register split (G = 3): producers dec to PREG, consumers inc to CREG <= 128 + (128 - PREG)
// * 128 / 384.  A/B: 24/160 (the producer loop spills a few bytes) for every family: config 3
// +1..3 %, config 4 +4 %, config 2 (two n = 32 units per warp) +2 % over 40/152.
template <class F>
struct Regs {
#ifdef VCA_PREG
    static constexpr int P = VCA_PREG;
#else
    static constexpr int P = F::G >= 3 ? 24 : 40;
#endif
#ifdef VCA_CREG
    static constexpr int C = VCA_CREG;
#else
    // G = 4: the launch pool is 640 threads x 96 registers, so 128 x 24 + 512 x C <= 61440
    static constexpr int C = F::G == 2 ? 232 : F::G == 3 ? 160 : 112;
#endif
};
constexpr int kConsumers = 4;

template <class F>
struct Lay {  // shared-memory layout (offsets from the 1024-aligned base)
    // ring + full/empty barriers + per-stage header words (VCA_DYN item index)
    static constexpr int GRP = (F::STAGES * F::STAGE + 2 * F::STAGES * 8 + F::STAGES * 4 + 1023) / 1024 * 1024;
    static constexpr int WTAB_OFF = F::GV * GRP;
    static constexpr int STASH_OFF = WTAB_OFF + (F::WTAB ? 32 * 32 * 8 : 0);
    static constexpr int WSM_OFF = STASH_OFF + 4 * F::GV * F::STASH;
    static constexpr int SMEM = 1024 + WSM_OFF + F::GV * 10 * 32 * 8;
    static_assert(SMEM <= 232448, "dynamic shared memory over the 227 KB per-CTA limit");
};

template <int W_, int BD_, int LP_, bool DUMP>
__global__ void __launch_bounds__(Fam<W_, BD_, LP_>::THREADS, Fam<W_, BD_, LP_>::G ? 1 : Fam<W_, BD_, LP_>::MINB) fused_kernel(const __grid_constant__ CUtensorMap tmY,
                                                    const __grid_constant__ CUtensorMap tmU,
                                                    const __grid_constant__ CUtensorMap tmV, const FusedArgs a)
{
    using F = Fam<W_, BD_, LP_>;
    constexpr int NY = F::NY, NC = F::NC, W = F::W, WC = F::WC, NU = F::NU;
    constexpr int kGroups = F::G, kGv = F::GV;
    uint8_t *smem_raw = vca_dyn_smem;
    using Y = Lay<F>;
    uint8_t *smem0p = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double *wtab = reinterpret_cast<double *>(smem0p + Y::WTAB_OFF);
    // per consumer warp: hst[32 slots][9] (8 row-group partials, padded) + sxs[32][4] DC sums
    uint8_t *stash = smem0p + Y::STASH_OFF;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // consumer group of this warp (producer warp g < kGroups feeds group g)
    const int grp = kGroups ? (warp < 4 ? warp : (warp >> 2) - 1) : 0;
    uint8_t *smem = smem0p + (grp < kGv ? grp : 0) * Y::GRP;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + F::STAGES * F::STAGE);
    uint64_t *empty = full + F::STAGES;
    const int vblk = blockIdx.x * kGv + grp, vgrid = gridDim.x * kGv;  // virtual CTA of the group
    if (threadIdx.x == 0) {
        for (int q = 0; q < kGv; ++q) {
            uint64_t *fq = reinterpret_cast<uint64_t *>(smem0p + q * Y::GRP + F::STAGES * F::STAGE);
            for (int i = 0; i < F::STAGES; ++i) {
                mbar_init(&fq[i], 1);
                mbar_init(&fq[F::STAGES + i], kConsumers);
            }
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (F::WTAB) {
        // luma n = 32 weights in [slot pair][lane][2] order (one conflict-free LDS.128 per pair):
        // slot = (mt*4 + r)*4 + e = 2 * pair + (e & 1), lane (g, t): i = 16mt + g + 8(e>>1),
        // j = 8r + 2t + (e&1)
        const double *W32 = a.W_all + table_offset(32);
        for (int idx = threadIdx.x; idx < 32 * 32; idx += blockDim.x) {
            const int ln = (idx >> 1) & 31, gg = ln >> 2, tt = ln & 3;
            const int slot = 2 * (idx >> 6) + (idx & 1);
            const int e = slot & 3, r = (slot >> 2) & 3, mt = slot >> 4;
            const int i = 16 * mt + gg + 8 * (e >> 1), j = 8 * r + 2 * tt + (e & 1);
            wtab[idx] = W32[i * 32 + j];
        }
    }
    __syncthreads();

    const int rows = a.rows, cols = a.cols;
    const int strips = (cols + F::UNITS - 1) / F::UNITS;
    const int items = a.n_frames * rows;  // < 2^31 (checked on the host)

    if (kGroups ? warp < 4 : warp == 0) {
        // ---------------- TMA producer (A1)
        if constexpr (kGroups != 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Regs<F>::P));
        if (lane == 0 && warp < kGv) {
            uint64_t policy;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmY)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmU)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmV)) : "memory");
            uint32_t st = 0, phase = 0;
            bool first_pass = true;
#if VCA_DYN
            int *hdr = reinterpret_cast<int *>(empty + F::STAGES);
            for (;;) {
                const unsigned long long tk = atomicAdd(a.ticket, 1ull) - a.ticket_base;
                const int it = tk < (unsigned long long)items ? (int)tk : -1;
                if (!first_pass) mbar_wait(smem_u32(&empty[st]), phase ^ 1);
                hdr[st] = it;  // published by the arrive below (release), read after the consumers' wait
                if (it < 0) {
                    mbar_arrive(smem_u32(&full[st]));  // end marker: a stage with no data
                    break;
                }
                const int f = it / rows, r = it - f * rows;
                for (int s = 0; s < strips; ++s) {
                    if (s > 0 && !first_pass) mbar_wait(smem_u32(&empty[st]), phase ^ 1);
                    uint8_t *base = smem + st * F::STAGE;
                    mbar_expect_tx(&full[st], F::TX);
                    if (a.y4) {
                        tma_load_4d(base, &tmY, &full[st], s * F::NBOX_Y, r * W, f, policy);
                    } else {
#pragma unroll
                        for (int b = 0; b < F::NBOX_Y; ++b)
                            tma_load_3d(base + b * F::BOXB_Y, &tmY, &full[st], (s * F::UNITS + b * F::UPB_Y) * W,
                                        r * W, f, policy);
                    }
                    if (a.c4) {
                        tma_load_4d(base + F::ST_Y, &tmU, &full[st], s * F::NBOX_C, r * WC, f, policy);
                        tma_load_4d(base + F::ST_Y + F::ST_C, &tmV, &full[st], s * F::NBOX_C, r * WC, f, policy);
                    } else {
#pragma unroll
                        for (int b = 0; b < F::NBOX_C; ++b) {
                            tma_load_3d(base + F::ST_Y + b * F::BOXB_C, &tmU, &full[st],
                                        (s * F::UNITS + b * F::UPB_C) * WC, r * WC, f, policy);
                            tma_load_3d(base + F::ST_Y + F::ST_C + b * F::BOXB_C, &tmV, &full[st],
                                        (s * F::UNITS + b * F::UPB_C) * WC, r * WC, f, policy);
                        }
                    }
                    if (++st == F::STAGES) {
                        st = 0;
                        phase ^= 1;
                        first_pass = false;
                    }
                }
            }
            (void)vblk;
            (void)vgrid;
#else
            // prefetch cursor VCA_L2PF strips ahead of the load cursor (same item sequence)
            int pit = vblk, ps = 0;
            if (VCA_L2PF > 0) {
                for (int k = 0; k < VCA_L2PF && pit < items; ++k)
                    if (++ps == strips) {
                        ps = 0;
                        pit += vgrid;
                    }
            }
            for (int it = vblk; it < items; it += vgrid) {
                const int f = it / rows, r = it - f * rows;
                for (int s = 0; s < strips; ++s) {
                    if (VCA_L2PF > 0 && pit < items) {
                        const int pf = pit / rows, pr = pit - pf * rows;
#pragma unroll
                        for (int b = 0; b < F::NBOX_Y; ++b)
                            tma_prefetch_3d(&tmY, (ps * F::UNITS + b * F::UPB_Y) * W, pr * W, pf);
#pragma unroll
                        for (int b = 0; b < F::NBOX_C; ++b) {
                            tma_prefetch_3d(&tmU, (ps * F::UNITS + b * F::UPB_C) * WC, pr * WC, pf);
                            tma_prefetch_3d(&tmV, (ps * F::UNITS + b * F::UPB_C) * WC, pr * WC, pf);
                        }
                        if (++ps == strips) {
                            ps = 0;
                            pit += vgrid;
                        }
                    }
                    if (!first_pass) mbar_wait(smem_u32(&empty[st]), phase ^ 1);
                    uint8_t *base = smem + st * F::STAGE;
#ifdef VCA_NULL_MEMORY
                    // compute-side probe (A/B only): release the stage without loading it --
                    // the consumers' own ceiling on whatever the ring holds
                    mbar_arrive(smem_u32(&full[st]));
                    (void)base;
                    if (++st == F::STAGES) {
                        st = 0;
                        phase ^= 1;
                        first_pass = false;
                    }
                    continue;
#endif
                    mbar_expect_tx(&full[st], F::TX);
                    if (a.y4) {
                        tma_load_4d(base, &tmY, &full[st], s * F::NBOX_Y, r * W, f, policy);
                    } else {
#pragma unroll
                        for (int b = 0; b < F::NBOX_Y; ++b)
                            tma_load_3d(base + b * F::BOXB_Y, &tmY, &full[st], (s * F::UNITS + b * F::UPB_Y) * W,
                                        r * W, f, policy);
                    }
                    if (a.c4) {
                        tma_load_4d(base + F::ST_Y, &tmU, &full[st], s * F::NBOX_C, r * WC, f, policy);
                        tma_load_4d(base + F::ST_Y + F::ST_C, &tmV, &full[st], s * F::NBOX_C, r * WC, f, policy);
                    } else {
#pragma unroll
                        for (int b = 0; b < F::NBOX_C; ++b) {
                            tma_load_3d(base + F::ST_Y + b * F::BOXB_C, &tmU, &full[st],
                                        (s * F::UNITS + b * F::UPB_C) * WC, r * WC, f, policy);
                            tma_load_3d(base + F::ST_Y + F::ST_C + b * F::BOXB_C, &tmV, &full[st],
                                        (s * F::UNITS + b * F::UPB_C) * WC, r * WC, f, policy);
                        }
                    }
                    if (++st == F::STAGES) {
                        st = 0;
                        phase ^= 1;
                        first_pass = false;
                    }
                }
            }
#endif
        }
        return;
    }

    // ---------------- consumers
    if constexpr (kGroups != 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Regs<F>::C));
    const int u = kGroups ? (warp & 3) : warp - 1;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t hst = smem_off(stash) + (grp * 4 + u) * F::STASH;  // [32][HW] doubles
    const uint32_t sxs = hst + 32 * F::HW * 8;             // [32][4] uint32
    // this lane's H partial slot within a unit's stash row (-1: the lane does not store)
    const bool hst_lane = F::HSLOTS == 8 ? t == 0 : (t & 1) == 0;
    const int hst_col = F::HSLOTS == 8 ? g : 2 * g + (t >> 1);
    UnitCtx<F> U;
    build_lane_const(U.L, a.T_all, g, t, NY);
    // per-lane scaled weights (A5): luma n = 16 positions (i = g + 8(e>>1), j = 8p + 2t + (e&1)),
    // chroma positions of dct16 (NC = 16) or dct8pair (NC = 8)
    {
        const double *W16 = a.W_all + table_offset(16);
        const double *W8 = a.W_all + table_offset(8);
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                U.wl16[p * 4 + e] = __ldg(W16 + (g + 8 * (e >> 1)) * 16 + 8 * p + 2 * t + (e & 1));
#pragma unroll
        for (int e = 0; e < UnitCtx<F>::NWC; ++e)
            U.wc[e] = NC == 16 ? U.wl16[e] : __ldg(W8 + g * 8 + 2 * t + e);
        const double *W4 = a.W_all + table_offset(4);
#pragma unroll
        for (int e = 0; e < 2; ++e) U.w4[e] = __ldg(W4 + (g & 3) * 4 + 2 * (t & 1) + e);
    }
    U.wtab = smem_off(wtab) + lane * 16;
    {
        // [e][lane] weight table (same values as the registers; filled by consumer warp 0)
        const uint32_t wsm0 = smem_off(smem0p + Y::WSM_OFF) + grp * 10 * 32 * 8;
        if (u == 0) {
#pragma unroll
            for (int e = 0; e < 8; ++e) sts<double>(wsm0 + (e * 32 + lane) * 8, U.wl16[e]);
#pragma unroll
            for (int e = 0; e < 2; ++e) sts<double>(wsm0 + ((8 + e) * 32 + lane) * 8, NC == 8 ? U.wc[e] : 0.0);
        }
        U.wsm = wsm0 + lane * 8;
        asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");  // this group's consumer warps
    }
    U.g = g;
    U.t = t;
    const double invNY = 1.0 / NY, invNC = 1.0 / NC;
    const uint32_t smem0 = smem_off(smem);  // stage boxes: data offsets
    const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
    const int64_t CY = (int64_t)rows * cols;
    uint64_t keep = 0;
#if VCA_EVICT_LAST
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
#endif

    // per-warp constants: smem offsets of this warp's units inside a stage, and the number of
    // leading strips in which all NU units of this warp are whole (valid, not a partial
    // last block column) -- those take the NU-wide fast path
    uint32_t offY[NU], offU[NU];
    int ubYc[NU], ubCc[NU];
#pragma unroll
    for (int n = 0; n < NU; ++n) {
        const int v = u + 4 * n;
        offY[n] = (v / F::UPB_Y) * F::BOXB_Y;
        offU[n] = F::ST_Y + (v / F::UPB_C) * F::BOXB_C;
        ubYc[n] = v % F::UPB_Y;
        ubCc[n] = v % F::UPB_C;
    }
    // NY = 8 lane geometry: the unit this lane loads for luma pair p (units 2p | 2p + 1, lane
    // t < 2 -> first) and for the 8-block chroma MMA (unit t, plane g >> 2)
    constexpr int M8 = NY == 8 ? NU / 4 : 1;  // 4-unit groups per warp per strip
    uint32_t LYoff[M8][2], LCoff[M8];
    int LYub[M8][2], LCub[M8];
#pragma unroll
    for (int m = 0; m < M8; ++m) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int v = u + 4 * (4 * m + 2 * p + (t >> 1));
            LYoff[m][p] = (v / F::UPB_Y) * F::BOXB_Y;
            LYub[m][p] = v % F::UPB_Y;
        }
        const int v = u + 4 * (4 * m + t);
        LCoff[m] = F::ST_Y + (v / F::UPB_C) * F::BOXB_C + (g >= 4 ? F::ST_C : 0);
        LCub[m] = v % F::UPB_C;
    }
    const int cols_whole = (a.width[0] % W) ? cols - 1 : cols;
    const int last_c = u + 4 * (NU - 1);  // c of this warp's last unit in strip 0
    const int s_fast = cols_whole > last_c ? (cols_whole - last_c - 1) / F::UNITS + 1 : 0;

    uint32_t st = 0, phase = 0;
#ifdef VCA_TIMES
    if (u == 0 && lane == 0 && vblk < 4096) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        vca_group_t[0][vblk] = gtimer();
        vca_group_t[2][vblk] = smid;
    }
#endif
#if VCA_DYN
    const uint32_t hdr0 = smem_off(empty + F::STAGES);
    for (;;) {
        mbar_wait(full0 + 8 * st, phase);  // the item's first stage, or the end marker
        const int it = lds<int>(hdr0 + 4 * st);
        if (it < 0) break;
#else
    for (int it = vblk; it < items; it += vgrid) {
#endif
        const int f = it / rows, r = it - f * rows;
        const int hvY = min(W, a.height[0] - r * W), hvC = min(WC, a.height[1] - r * WC);
        double hu = 0.0, hv = 0.0;                          // per-lane U/V texture partials (fixed order)
        ChromaAcc<F> ca;                                    // exact per-position chroma |C| sums
#pragma unroll
        for (int e = 0; e < ChromaAcc<F>::NP; ++e) ca.u[e] = ca.v[e] = 0u;
        // item sums of the flushed units' H_Y and L: warp totals in every lane, or (VCA_XRED8) per-lane
        // running sums reduced across lanes once at the item end
        double sHY = 0.0, sLY = 0.0, sLU = 0.0, sLV = 0.0;
        double *HYrow = a.s.HY + (int64_t)f * CY + (int64_t)r * cols;
        const int64_t fCY = (int64_t)f * CY;  // global index of the frame's first block (test outputs)
        // strips in chroma-flush windows of SPC: the flush runs once after each window (as its
        // own block, not if-converted into predicated instructions issued on every strip:
        // config 3 +1 %, config 4 +3.5 %, w = 16 full +7 %).  The n = 8 families keep the
        // in-loop flush (the windowed loop measured -3 % there).
        constexpr int SPC = ChromaAcc<F>::FC / NU;  // strips per chroma flush (<= FC units)
        static_assert(SPC >= 1, "chroma flush period");
        constexpr bool WIN = NY != 8;
        constexpr int SPCW = WIN ? SPC : (1 << 30);
        for (int s0 = 0; s0 < strips; s0 += SPCW) {
        const int s1 = min(strips, s0 + SPCW);
        for (int s = s0; s < s1; ++s) {
            if (!VCA_DYN || s > 0) mbar_wait(full0 + 8 * st, phase);
            // this warp's units of strip s: c_n = s*UNITS + u + 4n, n < NU, in ascending order;
            // unit m = s*NU + n of the item goes to stash slot m & 31
            const uint32_t base = smem0 + st * F::STAGE;
            const int c0 = s * F::UNITS + u;
#ifdef VCA_NULL_COMPUTE
            // memory-pipeline probe (A/B only): consumers touch one word of the stage and
            // release it -- the TMA ring's own ceiling for this layout
            if (lds32(base + 4 * lane) == 0xFFFFFFFFu && lane == 32) sHY += 1.0;
#else
            UnitOut o[NU];
            if (NY == 8) {
                // n = 8 families: always the 4-unit group path (whole strips without clamps)
                const uint32_t sl0 = (uint32_t)((s % F::SPF) * NU);
#pragma unroll
                for (int m = 0; m < M8; ++m) {
                    const int cm = c0 + 16 * m;  // column of the group's first unit
                    double hY4[4];
                    int32_t dY[4], dC[2];
                    int64_t kk[4];
#pragma unroll
                    for (int n = 0; n < 4; ++n)
                        kk[n] = ((DUMP || kMutate) && cm + 4 * n < cols) ? fCY + (int64_t)r * cols + cm + 4 * n : -1;
                    if (s < s_fast) {
                        const int wY[2] = {W, W};
                        process_group8<F, false, DUMP>(U, a, base, LYoff[m], LYub[m], LCoff[m], LCub[m], hvY, hvC, wY,
                                                       WC, kk, hY4, dY, dC, ca);
                    } else {
                        // valid width of the unit this lane loads; units past the last column read
                        // the zero-filled box unclamped (never stored)
                        int wY[2];
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            const int c = cm + 4 * (2 * p + (t >> 1));
                            wY[p] = c < cols ? min(W, a.width[0] - c * W) : W;
                        }
                        const int cC = cm + 4 * t;
                        const int wC = cC < cols ? min(WC, a.width[1] - cC * WC) : WC;
                        process_group8<F, true, DUMP>(U, a, base, LYoff[m], LYub[m], LCoff[m], LCub[m], hvY, hvC, wY,
                                                      wC, kk, hY4, dY, dC, ca);
                    }
                    const uint32_t slm = sl0 + 4 * m;
#pragma unroll
                    for (int n = 0; n < 4; ++n) {
                        if (t == 0) sts<double>(hst + ((slm + n) * F::HW + g) * 8, hY4[n]);
                        if (lane == 0) sts<uint32_t>(sxs + (slm + n) * 16, (uint32_t)dY[n]);
                    }
                    if ((g & 3) == 0 && (t & 1) == 0) {  // chroma DCs: units t >> 1 and 2 + (t >> 1), plane g >> 2
                        sts<uint32_t>(sxs + (slm + (t >> 1)) * 16 + 4 * (1 + (g >> 2)), (uint32_t)dC[0]);
                        sts<uint32_t>(sxs + (slm + 2 + (t >> 1)) * 16 + 4 * (1 + (g >> 2)), (uint32_t)dC[1]);
                    }
                }
            } else if (s < s_fast) {
                uint32_t bY[NU], bU[NU];
                int64_t kk[NU];
#pragma unroll
                for (int n = 0; n < NU; ++n) {
                    bY[n] = base + offY[n];
                    bU[n] = base + offU[n];
                    kk[n] = (DUMP || kMutate) ? fCY + (int64_t)r * cols + c0 + 4 * n : 0;
                }
                process_units<F, false, DUMP, NU>(U, a, bY, bU, ubYc, ubCc, hvY, hvC, W, WC, kk, o, hu, hv, ca);
                // stash: per-unit luma row-group partials and raw C_00 values, reduced SPF strips
                // (<= 32 units) at a time
                const uint32_t sl0 = (uint32_t)((s % F::SPF) * NU);
#pragma unroll
                for (int n = 0; n < NU; ++n) {
                    if (hst_lane) sts<double>(hst + ((sl0 + n) * F::HW + hst_col) * 8, o[n].hY);
                    if (lane == 0) sts<uint4>(sxs + (sl0 + n) * 16, make_uint4(o[n].dcY, o[n].dcU, o[n].dcV, 0u));
                }
            } else {
                // ragged strip end or a partial last block column: whole units 0 and 1 of this
                // warp (if any) as one 2-unit group, the rest one unit at a time
                int n0 = 0;
                if (VCA_RAGGED2 && NU >= 4 && c0 + 4 < cols_whole) {
                    uint32_t bY[2], bU[2];
                    int uY[2], uC[2];
                    int64_t kk[2];
#pragma unroll
                    for (int n = 0; n < 2; ++n) {
                        bY[n] = base + offY[n];
                        bU[n] = base + offU[n];
                        uY[n] = ubYc[n];
                        uC[n] = ubCc[n];
                        kk[n] = fCY + (int64_t)r * cols + c0 + 4 * n;
                    }
                    UnitOut o2[2];
                    process_units<F, false, DUMP, 2>(U, a, bY, bU, uY, uC, hvY, hvC, W, WC, kk, o2, hu, hv, ca);
                    const uint32_t sl0 = (uint32_t)((s % F::SPF) * NU);
#pragma unroll
                    for (int n = 0; n < 2; ++n) {
                        if (hst_lane) sts<double>(hst + ((sl0 + n) * F::HW + hst_col) * 8, o2[n].hY);
                        if (lane == 0)
                            sts<uint4>(sxs + (sl0 + n) * 16, make_uint4(o2[n].dcY, o2[n].dcU, o2[n].dcV, 0u));
                    }
                    n0 = 2;
                }
#pragma unroll
                for (int n = 0; n < NU; ++n) {
                    const int c = c0 + 4 * n;
                    if (n < n0 || c >= cols) continue;
                    const int v = u + 4 * n;
                    const uint32_t bY[1] = {base + (v / F::UPB_Y) * F::BOXB_Y};
                    const uint32_t bU[1] = {base + F::ST_Y + (v / F::UPB_C) * F::BOXB_C};
                    const int uY[1] = {v % F::UPB_Y}, uC[1] = {v % F::UPB_C};
                    const int64_t kk[1] = {fCY + (int64_t)r * cols + c};
                    const int wvY = min(W, a.width[0] - c * W), wvC = min(WC, a.width[1] - c * WC);
                    UnitOut o1[1];
                    if (wvY < W)
                        process_units<F, true, DUMP, 1>(U, a, bY, bU, uY, uC, hvY, hvC, wvY, wvC, kk, o1, hu, hv, ca);
                    else
                        process_units<F, false, DUMP, 1>(U, a, bY, bU, uY, uC, hvY, hvC, W, WC, kk, o1, hu, hv, ca);
                    const uint32_t slot = (uint32_t)((s % F::SPF) * NU + n);
                    if (hst_lane) sts<double>(hst + (slot * F::HW + hst_col) * 8, o1[0].hY);
                    if (lane == 0) sts<uint4>(sxs + slot * 16, make_uint4(o1[0].dcY, o1[0].dcU, o1[0].dcV, 0u));
                }
            }
#endif
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * st);
            if (++st == F::STAGES) {
                st = 0;
                phase ^= 1;
            }
            if (!WIN && ChromaAcc<F>::ON && ((s % SPC) == SPC - 1 || s == strips - 1)) {
#pragma unroll
                for (int e = 0; e < ChromaAcc<F>::NP; ++e) {
                    const double wce = NY == 8 ? U.w4[e] : U.wc[e];
                    hu = fma(wce, __uint2double_rn(ca.u[e]), hu);
                    hv = fma(wce, __uint2double_rn(ca.v[e]), hv);
                    ca.u[e] = ca.v[e] = 0u;
                }
            }
            if ((s % F::SPF) == F::SPF - 1 || s == strips - 1) {
                // flush: lane l finishes unit m = first unit of the window + l -- H_Y (fixed
                // order over the 8 row groups), its L terms (A6), the per-block H_Y store (A5,
                // needed for h); then a fixed xor tree over lanes into the running item sums.
                const int nwin = ((s % F::SPF) + 1) * NU;  // units stashed in this window
                const int m = (s - (s % F::SPF)) * NU + lane;
                const int cl = (m / NU) * F::UNITS + u + 4 * (m % NU);
                double Hl = 0.0, LYl = 0.0, LUl = 0.0, LVl = 0.0;
                if (lane < nwin && cl < cols) {
#pragma unroll
                    for (int gg = 0; gg < F::HSLOTS; ++gg) Hl += lds_f64(hst + (lane * F::HW + gg) * 8);
                    // A6: sum x = C_00 / 4096 exactly (C_00 mod 2^32 suffices: sum x < 2^20, R-11)
                    const uint4 dc = lds<uint4>(sxs + lane * 16);
                    LYl = sqrt((double)(dc.x >> 12) * invNY);
                    LUl = sqrt((double)(dc.y >> 12) * invNC);
                    LVl = sqrt((double)(dc.z >> 12) * invNC);
#ifdef VCA_DEBUG_BOUNDS
                    if (cl < 0 || cl >= cols) __trap();
#endif
                    st_keep(HYrow + cl, Hl, keep);
                }
                if (!VCA_XRED8) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        Hl += __shfl_xor_sync(0xffffffffu, Hl, o);
                        LYl += __shfl_xor_sync(0xffffffffu, LYl, o);
                        LUl += __shfl_xor_sync(0xffffffffu, LUl, o);
                        LVl += __shfl_xor_sync(0xffffffffu, LVl, o);
                    }
                }
                sHY += Hl;
                sLY += LYl;
                sLU += LUl;
                sLV += LVl;
                __syncwarp();
            }
        }
        if (WIN && ChromaAcc<F>::ON) {
            // chroma flush: weight the exact per-position sums once (fixed position order)
#pragma unroll
            for (int e = 0; e < ChromaAcc<F>::NP; ++e) {
                const double wce = NY == 8 ? U.w4[e] : U.wc[e];
                hu = fma(wce, __uint2double_rn(ca.u[e]), hu);
                hv = fma(wce, __uint2double_rn(ca.v[e]), hv);
                ca.u[e] = ca.v[e] = 0u;
            }
        }
        }
        // ---- item end: fixed-order partials of this warp's units (A7 inputs)
        if (VCA_XRED8) {
            // value r = {H_Y, L_Y, H_U, L_U, H_V, L_V}: lane 4 r stores the warp total of value r
            const double vals[8] = {sHY, sLY, hu, sLU, hv, sLV, 0.0, 0.0};
            const double tot = xred8(vals, lane);
            const int r6 = lane >> 2;
            if ((lane & 3) == 0 && r6 < 6) {
                const int64_t q = (int64_t)r * kConsumers + u;
                double *P = a.s.partial + (((int64_t)f * 3 + (r6 >> 1)) * a.s.P + q) * 2 + (r6 & 1);
                st_keep(P, tot, keep);
            }
        } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            hu += __shfl_xor_sync(0xffffffffu, hu, o);
            hv += __shfl_xor_sync(0xffffffffu, hv, o);
        }
        if (lane == 0) {
            const int64_t q = (int64_t)r * kConsumers + u;
            double *P0 = a.s.partial + (((int64_t)f * 3 + 0) * a.s.P + q) * 2;
            double *P1 = a.s.partial + (((int64_t)f * 3 + 1) * a.s.P + q) * 2;
            double *P2 = a.s.partial + (((int64_t)f * 3 + 2) * a.s.P + q) * 2;
            st_keep(P0, sHY, keep);
            st_keep(P0 + 1, sLY, keep);
            st_keep(P1, hu, keep);
            st_keep(P1 + 1, sLU, keep);
            st_keep(P2, hv, keep);
            st_keep(P2 + 1, sLV, keep);
        }
        }
    }
#ifdef VCA_TIMES
    if (u == 0 && lane == 0 && vblk < 4096) vca_group_t[1][vblk] = gtimer();
#endif
}

// ------------------------------------------------------------------ host side
inline bool fused_supported(int w, int lowpass, bool grids_equal)
{
    return grids_equal && (w == 32 || w == 16 || (w == 8 && !lowpass));
}
inline int fused_partials_per_row() { return 4; }

typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                    const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode()
{
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

#ifndef VCA_L2PROMO
#define VCA_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B  // A/B: NONE / L2_64B / L2_128B / L2_256B
#endif

inline bool make_map(CUtensorMap *m, const PlaneDesc &P, int n_frames, int es, int inner_bytes, int box_rows)
{
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)P.width, (cuuint64_t)P.height, (cuuint64_t)n_frames};
    cuuint64_t strides[2] = {(cuuint64_t)P.pitch, (cuuint64_t)(P.fstride > 0 ? P.fstride : P.pitch * P.height)};
    cuuint32_t box[3] = {(cuuint32_t)(inner_bytes / es), (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUtensorMapSwizzle sw = inner_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : inner_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = enc(m, es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                     const_cast<uint8_t *>(P.base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     VCA_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int W, int BD, int LP>
inline cudaError_t prepare_one()
{
    using F = Fam<W, BD, LP>;
    cudaError_t e = cudaFuncSetAttribute(fused_kernel<W, BD, LP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Lay<F>::SMEM);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fused_kernel<W, BD, LP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay<F>::SMEM);
    return e;
}

inline cudaError_t fused_prepare(int bd, int lowpass, int w)
{
    if (w == 32 && lowpass) return bd == 8 ? prepare_one<32, 8, 1>() : prepare_one<32, 10, 1>();
    if (w == 32) return bd == 8 ? prepare_one<32, 8, 0>() : prepare_one<32, 10, 0>();
    if (w == 16 && lowpass) return bd == 8 ? prepare_one<16, 8, 1>() : prepare_one<16, 10, 1>();
    if (w == 8) return bd == 8 ? prepare_one<8, 8, 0>() : prepare_one<8, 10, 0>();
    return bd == 8 ? prepare_one<16, 8, 0>() : prepare_one<16, 10, 0>();
}

template <int W, int BD, int LP>
inline int launch_one(const Planes3 &pl, int n_frames, const int8_t *T, const double *Wt, const Scratch &s,
                      const DumpPtrs &dp, int sm_count, cudaStream_t st, unsigned long long *ticket,
                      unsigned long long *ticket_base)
{
    using F = Fam<W, BD, LP>;
    CUtensorMap mY, mU, mV;
    int y4 = 0, u4 = 0, v4 = 0;
    if (!make_plane_map(&mY, pl.p[0], n_frames, F::ES, F::IB_Y, W, F::NBOX_Y, &y4) ||
        !make_plane_map(&mU, pl.p[1], n_frames, F::ES, F::IB_C, W / 2, F::NBOX_C, &u4) ||
        !make_plane_map(&mV, pl.p[2], n_frames, F::ES, F::IB_C, W / 2, F::NBOX_C, &v4))
        return -2;
    if (u4 != v4 && !make_map(u4 ? &mU : &mV, u4 ? pl.p[1] : pl.p[2], n_frames, F::ES, F::IB_C, W / 2))
        return -2;  // (U and V share one flag; equal geometry makes this unreachable)
    FusedArgs a;
    a.y4 = y4;
    a.c4 = u4 && v4;
    a.n_frames = n_frames;
    for (int p = 0; p < 3; ++p) {
        a.width[p] = pl.p[p].width;
        a.height[p] = pl.p[p].height;
    }
    a.cols = pl.p[0].cols;
    a.rows = pl.p[0].rows;
    a.W_all = Wt;
    a.T_all = T;
    a.s = s;
    a.dump = dp;
    a.ticket = ticket;
    a.ticket_base = ticket_base ? *ticket_base : 0;
    const bool dump = dp.on != 0;
    auto kern = dump ? fused_kernel<W, BD, LP, true> : fused_kernel<W, BD, LP, false>;
    // CTAs per SM: a property of the kernel and the device, queried once per instantiation
    // (the query costs microseconds of host time on every call otherwise)
    static std::atomic<int> cached[2] = {0, 0};
    int per_sm = cached[dump].load(std::memory_order_relaxed);
    if (per_sm < 1) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, F::THREADS, Lay<F>::SMEM) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        cached[dump].store(per_sm, std::memory_order_relaxed);
    }
    const int64_t items = (int64_t)n_frames * a.rows;
    if (items > 0x7fffffff) return -2;
    int64_t grid = (int64_t)sm_count * per_sm;
    if (grid > items) grid = items;
    kern<<<(unsigned)grid, F::THREADS, Lay<F>::SMEM, st>>>(mY, mU, mV, a);
    // every group takes exactly one ticket past the last item: the next launch starts after them
    if (ticket_base) *ticket_base += (unsigned long long)items + (unsigned long long)grid * F::GV;
    return 0;
}

// 4-D map of a plane (bytes within a box row, rows, box index along the row, frame): one TMA loads a
// strip's nb boxes into the same smem layout as nb 3-D loads.  Used when every box is whole (row
// bytes a multiple of the box width: no box reads past a row) and boxes have >= 8 rows (the smem
// box stride of the 4-row chroma boxes of the w = 8 family is padded to 8 rows).
inline bool map4_ok(const PlaneDesc &P, int es, int inner_bytes, int box_rows, int nb)
{
    return VCA_TMA4 && nb > 1 && box_rows >= 8 && ((int64_t)P.width * es) % inner_bytes == 0;
}

inline bool make_map4(CUtensorMap *m, const PlaneDesc &P, int n_frames, int es, int inner_bytes, int box_rows, int nb)
{
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)(inner_bytes / es), (cuuint64_t)P.height,
                          (cuuint64_t)(((int64_t)P.width * es) / inner_bytes), (cuuint64_t)n_frames};
    cuuint64_t strides[3] = {(cuuint64_t)P.pitch, (cuuint64_t)inner_bytes,
                             (cuuint64_t)(P.fstride > 0 ? P.fstride : P.pitch * P.height)};
    cuuint32_t box[4] = {(cuuint32_t)(inner_bytes / es), (cuuint32_t)box_rows, (cuuint32_t)nb, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUtensorMapSwizzle sw = inner_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : inner_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = enc(m, es == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4,
                     const_cast<uint8_t *>(P.base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     VCA_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// the plane's map: 4-D when map4_ok and encodable, else 3-D; *four says which
inline bool make_plane_map(CUtensorMap *m, const PlaneDesc &P, int n_frames, int es, int inner_bytes, int box_rows,
                           int nb, int *four)
{
    if (map4_ok(P, es, inner_bytes, box_rows, nb) && make_map4(m, P, n_frames, es, inner_bytes, box_rows, nb)) {
        *four = 1;
        return true;
    }
    *four = 0;
    return make_map(m, P, n_frames, es, inner_bytes, box_rows);
}

template <int W, int BD, int LP>
inline bool check_one(const Planes3 &pl, int n_frames)
{
    using F = Fam<W, BD, LP>;
    CUtensorMap m;
    return make_map(&m, pl.p[0], n_frames, F::ES, F::IB_Y, W) && make_map(&m, pl.p[1], n_frames, F::ES, F::IB_C, W / 2) &&
           make_map(&m, pl.p[2], n_frames, F::ES, F::IB_C, W / 2) && (int64_t)n_frames * pl.p[0].rows <= 0x7fffffff;
}

// True if launch_fused would accept these planes (tensor maps encodable, item count in range).
inline bool fused_check(const Planes3 &pl, int n_frames, int bd, int lowpass)
{
    const int w = pl.p[0].w;
    if (w == 32 && lowpass) return bd == 8 ? check_one<32, 8, 1>(pl, n_frames) : check_one<32, 10, 1>(pl, n_frames);
    if (w == 32) return bd == 8 ? check_one<32, 8, 0>(pl, n_frames) : check_one<32, 10, 0>(pl, n_frames);
    if (w == 16 && lowpass) return bd == 8 ? check_one<16, 8, 1>(pl, n_frames) : check_one<16, 10, 1>(pl, n_frames);
    if (w == 8) return bd == 8 ? check_one<8, 8, 0>(pl, n_frames) : check_one<8, 10, 0>(pl, n_frames);
    return bd == 8 ? check_one<16, 8, 0>(pl, n_frames) : check_one<16, 10, 0>(pl, n_frames);
}

// Returns 0 on launch, -1 on a CUDA launch failure (see cudaGetLastError), -2 if a
// tensor map could not be encoded.
inline int launch_fused(const Planes3 &pl, int n_frames, int bd, int lowpass, const int8_t *T, const double *Wt,
                        const Scratch &s, const DumpPtrs &dp, int sm_count, cudaStream_t st, unsigned long long *ticket,
                        unsigned long long *ticket_base)
{
    const int w = pl.p[0].w;
    if (w == 32 && lowpass)
        return bd == 8 ? launch_one<32, 8, 1>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base)
                       : launch_one<32, 10, 1>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base);
    if (w == 32)
        return bd == 8 ? launch_one<32, 8, 0>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base)
                       : launch_one<32, 10, 0>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base);
    if (w == 16 && lowpass)
        return bd == 8 ? launch_one<16, 8, 1>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base)
                       : launch_one<16, 10, 1>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base);
    if (w == 8)
        return bd == 8 ? launch_one<8, 8, 0>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base)
                       : launch_one<8, 10, 0>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base);
    return bd == 8 ? launch_one<16, 8, 0>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base)
                   : launch_one<16, 10, 0>(pl, n_frames, T, Wt, s, dp, sm_count, st, ticket, ticket_base);
}

}  // namespace vca
