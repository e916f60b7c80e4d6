/*
 * vca.h -- C ABI of libvca, the B200 (sm_100a) hot path of the Video
 * Complexity Analyzer v2.0 (arxiv 2304.12384).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, R-k = DESIGN.md
 * reading k.  The operation (section 2 "Video complexity analyzer"):
 * for every frame of 8/10-bit 4:2:0 video, per block of the Y, U and V
 * planes, an exact integer 2-D DCT (R-1) -- optionally of the 2x2
 * low-pass-downsampled block (R-5) -- reduced to the texture energy
 * H = sum_{(i,j)!=(0,0)} w_n(i,j) |C_ij| / (4096 n) (R-2, R-3)
 * and the luminescence sqrt(C_00 / (4096 n)), averaged per
 * frame into E_Y, L_Y, E_U, L_U, E_V, L_V, plus the luma
 * gradient h = sum_k |H_t[k] - H_{t-1}[k]| / (C_Y n^2) (R-7).
 *
 * Conventions for every entry point:
 *  - Return value: VCA_OK (0) or a negative VCA_ERR_* code; nothing is
 *    thrown or aborted across the ABI.  An argument error leaves the context
 *    valid and unchanged.  A CUDA error poisons the context: every later
 *    call on it returns VCA_ERR_CUDA until vca_destroy.
 *  - Device pointers are CUDA device addresses on the current device; host
 *    pointers are plain host memory.  The caller owns every buffer passed in
 *    (planes, scratch, outputs); the context owns only its tables, its
 *    carried previous-frame state and (for vca_analyze_host) its staging.
 *  - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *    stream) and the call returns after launch; results are valid once the
 *    stream is synchronised.  A context must not be used from two threads
 *    at once, and its calls must execute in call order on the device (one
 *    stream, or streams ordered by events): each call reads the previous
 *    frame's energies the call before it left in the context (R-7).
 *  - Results are bit-identical for any split of a sequence into calls, any
 *    frame-range partition across GPUs (with a one-frame halo) and any
 *    launch configuration.
 */
#ifndef VCA_H
#define VCA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vca_ctx vca_ctx;

/* One per-frame record, 64 bytes, in the CSV column order of S:456:
 * POC,E_Y,h,L_Y,E_U,L_U,E_V,L_V.  All features >= 0; h = 0 at sequence
 * start. */
typedef struct {
    int64_t poc;
    double E_Y, h, L_Y, E_U, L_U, E_V, L_V;
} vca_features;

enum {
    VCA_OK = 0,
    VCA_ERR_INVALID_ARG = -1,
    VCA_ERR_UNSUPPORTED_BLOCK_SIZE = -2,
    VCA_ERR_UNSUPPORTED_BIT_DEPTH = -3,
    VCA_ERR_UNSUPPORTED_CHROMA = -4,
    VCA_ERR_GEOMETRY = -5,
    VCA_ERR_ALIGNMENT = -6,
    VCA_ERR_CUDA = -7,
    VCA_ERR_OOM = -8,
    VCA_ERR_SCRATCH = -9
};

enum { VCA_CHROMA_420 = 0, VCA_CHROMA_422 = 1, VCA_CHROMA_444 = 2 };

/* Kernel path the context resolved to (informational; there is one CUDA
 * backend, these are its two kernel families): the fused TMA + tensor-core kernel
 * for every block size whose chroma grid equals the luma grid (w = 8, 16, 32; w = 16
 * and 32 also low-pass), a CUDA-core kernel (one thread per 4x4 block) for w = 4. */
enum { VCA_PATH_FUSED_MMA = 1, VCA_PATH_WARP_GENERIC = 2 };

/* Resolved geometry of a context (vca_get_info). */
typedef struct {
    int width, height, bit_depth, lowpass;
    int block[3];      /* block size w per plane (Y, U, V) in samples, R-9       */
    int n[3];          /* DCT size per plane: w, or w/2 in low-pass (R-5)        */
    int cols[3];       /* ceil(plane_width / w)                                  */
    int rows[3];       /* ceil(plane_height / w)                                 */
    int64_t count[3];  /* C = cols * rows                                */
    int path;          /* VCA_PATH_*                                             */
} vca_info;

/* Create a context for one stream geometry.
 * width, height: luma size in samples; even (4:2:0), >= 2 (R-12).
 * bit_depth: 8 (uint8 samples) or 10 (little-endian uint16 containers,
 *   values > 1023 clamp to 1023, R-10); else VCA_ERR_UNSUPPORTED_BIT_DEPTH.
 * chroma_format: VCA_CHROMA_420 only; else VCA_ERR_UNSUPPORTED_CHROMA (R-9).
 * block_size: 0 (auto: 32 if height >= 2160, 16 if >= 1080, else 8)
 *   or 4, 8, 16, 32; else VCA_ERR_UNSUPPORTED_BLOCK_SIZE.  Chroma block =
 *   max(4, w/2).
 * lowpass: 0 or 1; requires chroma block >= 8, i.e. w >= 16, else
 *   VCA_ERR_UNSUPPORTED_BLOCK_SIZE (R-9).
 * The new context starts a sequence at POC 0.  Allocates the context's
 * device tables and carried state on the current device; VCA_ERR_OOM /
 * VCA_ERR_CUDA on failure.  *out is set only on success. */
int vca_create(int width, int height, int bit_depth, int chroma_format, int block_size, int lowpass,
               vca_ctx **out);

/* Fill *info with the resolved geometry.  VCA_ERR_INVALID_ARG on NULL. */
int vca_get_info(const vca_ctx *ctx, vca_info *info);

/* Bytes of device scratch vca_analyze needs for up to max_frames frames
 * per call (per-block luma energies and per-row partial sums).  0 on a NULL
 * context or max_frames < 1. */
size_t vca_scratch_bytes(const vca_ctx *ctx, int max_frames);

/* Analyse n_frames frames already resident in device memory.
 * planes[p]: device address of frame 0 of plane p (0 = Y, 1 = U, 2 = V);
 *   frame t of plane p starts at planes[p] + t * frame_stride_bytes[p];
 *   row y at + y * pitch_bytes[p].  Plane p is (width >> (p>0)) x
 *   (height >> (p>0)) samples of 1 (8-bit) or 2 (10-bit) bytes.
 * Requirements: non-NULL planes; pitch >= row bytes; planes, pitches and
 *   frame strides 16-byte aligned (VCA_ERR_ALIGNMENT otherwise).
 * n_halo: 0 or 1.  With 1, frame 0 only provides the previous-frame luma
 *   energies for frame 1 and emits no record (range start of a frame-range
 *   shard, R-7).  n_frames >= 1 + n_halo, else VCA_ERR_INVALID_ARG.
 * scratch / scratch_bytes: caller-owned device memory of at least
 *   vca_scratch_bytes(ctx, n_frames) bytes (VCA_ERR_SCRATCH otherwise),
 *   8-byte aligned; clobbered.  After the call (stream-ordered) it begins with
 *   the per-block luma energies H_Y (A5, the inputs of h) as doubles
 *   [n_frames][rows[0] * cols[0]] in raster block order -- the halo frame's too.
 * out_dev: device array of n_frames - n_halo records, written in POC order.
 *   Record i has poc = next_poc + i, where next_poc is the context's POC
 *   counter (0 after create; see vca_reset), advanced by n_frames - n_halo.
 *   h of the first emitted frame uses, in order of preference: the halo
 *   frame; the energies carried from the previous call on this context; 0
 *   at sequence start.
 * stream: cudaStream_t to enqueue on.  Launch errors -> VCA_ERR_CUDA. */
int vca_analyze(vca_ctx *ctx, const void *const planes[3], const int64_t pitch_bytes[3],
                const int64_t frame_stride_bytes[3], int n_frames, int n_halo, void *scratch,
                size_t scratch_bytes, vca_features *out_dev, void *stream);

/* End-to-end variant from HOST memory: the same operation as vca_analyze,
 * with planes in host memory (pinned memory gives full PCIe bandwidth; any
 * host memory works) and records written to host memory out_host.  Frames
 * are copied in chunks into context-owned device staging (allocated on the
 * first call, sized for chunk_frames frames, reused after) on `stream`,
 * with the copy of chunk k+1 overlapping the analysis of chunk k on an
 * internal stream pair.  Returns after the records are in out_host (the
 * call synchronises).  chunk_frames <= 0 selects 8.  Same requirements and
 * errors as vca_analyze (alignment applies to the host addresses too). */
int vca_analyze_host(vca_ctx *ctx, const void *const host_planes[3], const int64_t pitch_bytes[3],
                     const int64_t frame_stride_bytes[3], int n_frames, int n_halo, int chunk_frames,
                     vca_features *out_host, void *stream);

/* Start a new sequence: the next emitted frame gets POC next_poc and, unless
 * a halo precedes it, h = 0.  Enqueues nothing. */
int vca_reset(vca_ctx *ctx, int64_t next_poc);

/* Optional device-side timing (used by bench.py for the roofline): when
 * enabled, vca_analyze records CUDA events on `stream` around each kernel it
 * launches.  vca_profile_read synchronises those events and returns the
 * summed milliseconds of the block kernel (A1-A7) and of the per-frame
 * finalize kernel (A7-A9) since the last read, and the number of kernel
 * launches counted since the last read; then resets the sums. */
int vca_profile_enable(vca_ctx *ctx, int enable);
int vca_profile_read(vca_ctx *ctx, double *block_kernel_ms, double *finalize_ms, int64_t *launches);

/* TEST-ONLY: analyse the single frame whose planes start at device
 * addresses planes[0..2] (rows pitch_bytes[p] apart) with the DUMP
 * instantiation of this context's block kernel (the production kernel's
 * source with test outputs added; vca_debug_analyze ties its results to the
 * production instantiation bit for bit), and copy to host, for every plane p
 * with a non-NULL coeffs[p]: coeffs[p][k][i][j] (int32; C_00 is stored mod
 * 2^32, R-11) for every block k in raster order and, where the pointer is
 * non-NULL, sumx[p][k] (sum of the samples entering the DCT), H[p][k] and
 * L[p][k].  Host arrays hold count[p] * n[p]^2, count[p], count[p] and
 * count[p] entries.  Planes with a NULL coeffs[p] are not dumped.  The four
 * pointer arrays themselves must be non-NULL (VCA_ERR_INVALID_ARG).  Does not
 * touch the carried state.  Synchronises the device. */
int vca_debug_dump(vca_ctx *ctx, const void *const planes[3], const int64_t pitch_bytes[3],
                   int32_t *const coeffs[3], int64_t *const sumx[3], double *const H[3],
                   double *const L[3]);

/* TEST-ONLY: exactly vca_analyze (same arguments, records, scratch contents,
 * carried state and errors), run through the DUMP instantiation of the block
 * kernel, which additionally writes, for every block k of every frame t
 * (index t * count[p] + k) of every plane p whose pointer is non-NULL, into
 * caller-owned DEVICE arrays of n_frames * count[p] entries:
 *   chk_dev[p]:  sum over (i,j) != (0,0) of C_ij * (i * n[p] + j + 1), the
 *                exact AC checksum (int64, wrapping; the library zeroes the
 *                array first, on `stream`);
 *   sumx_dev[p]: sum of the DCT input samples (= C_00 / 4096, R-2);
 *   H_dev[p]:    the block's texture energy H (A5).
 * Records and scratch must equal vca_analyze's bit for bit on the same input
 * (tests/test_parity_gpu.py); the per-block integers pin every coefficient of
 * every block against the oracle (SURVEY 8(c) "Whole pipeline").  chk_dev,
 * sumx_dev and H_dev may be NULL, or hold NULL entries. */
int vca_debug_analyze(vca_ctx *ctx, const void *const planes[3], const int64_t pitch_bytes[3],
                      const int64_t frame_stride_bytes[3], int n_frames, int n_halo, void *scratch,
                      size_t scratch_bytes, vca_features *out_dev, int64_t *const chk_dev[3],
                      int64_t *const sumx_dev[3], double *const H_dev[3], void *stream);

/* TEST-ONLY (suite self-test): in a library built with -DVCA_MUTATE, add 1 to
 * coefficient pos = i * n + j ((i,j) != (0,0)) of block `block` (global index
 * t * count[plane] + k of the call) of plane `plane` in the kernel
 * instantiations selected by `which` (bit 0: production, bit 1: DUMP), for
 * every later launch in this process; plane -1 switches it off.  Returns
 * VCA_ERR_INVALID_ARG in every other build. */
int vca_debug_mutate(int plane, int64_t block, int pos, int which);

void vca_destroy(vca_ctx *ctx);

/* Static string for a status code. */
const char *vca_status_string(int status);

/* Library version string, "vca-b200 <major>.<minor>". */
const char *vca_version(void);

#ifdef __cplusplus
}
#endif

#endif /* VCA_H */
