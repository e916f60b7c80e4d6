// vca_api.cu -- host side of libvca: the C ABI declared in include/vca.h.
// Validation (R-9..R-12), geometry,
// basis / weight tables (R-1, R-3, generated here, independently of the
// oracle), the carried previous-frame state (R-7), launches on the caller's
// stream, the host-memory end-to-end pipeline, profiling and the test dump.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/vca.h"
#include "../../include/vca_io.h"
#include "kernel_finalize.cuh"
#include "kernel_fused.cuh"
#include "kernel_generic.cuh"
#include "vca_common.cuh"

using namespace vca;

namespace {

struct EventTriple {
    cudaEvent_t e[3];
};

}  // namespace

struct vca_ctx {
    int width = 0, height = 0, bd = 8, lowpass = 0;
    PlaneDesc geo[3];  // geometry only (base/pitch/fstride filled per call)
    int path = VCA_PATH_WARP_GENERIC;
    int P = 0, Pp[3] = {0, 0, 0};
    int device = 0, sm_count = 148;
    int8_t *d_T = nullptr;     // basis tables, all sizes
    double *d_W = nullptr;     // scaled weight tables, all sizes
    double *d_prevHY = nullptr;  // two buffers of C_Y doubles: [cur_prev] holds the carried H_Y
    unsigned long long *d_ticket = nullptr;  // dynamic item scheduling (VCA_DYN): never reset
    unsigned long long ticket_base = 0;      // first ticket of the next launch
    int cur_prev = 0;
    bool prev_valid = false;
    int64_t next_poc = 0;
    bool poisoned = false;
    // profiling
    bool prof = false;
    std::vector<EventTriple> pool, pending;
    double acc_block_ms = 0, acc_fin_ms = 0;
    int64_t launches = 0;
    // host end-to-end staging
    uint8_t *stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    int stage_frames = 0;
    void *h_scratch = nullptr;
    size_t h_scratch_bytes = 0;
    vca_features *d_rec = nullptr;
    size_t d_rec_n = 0;
    cudaStream_t s_copy = nullptr, s_comp = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
};

namespace {

#ifndef VCA_FIN_FRAMES
#define VCA_FIN_FRAMES 1  // max consecutive frames per finalize CTA (power of two; A/B: 2, 4 slower -- latency-bound chain)
#endif

int fail_cuda(vca_ctx *ctx, cudaError_t e)
{
    if (e != cudaSuccess) {
        if (ctx) ctx->poisoned = true;
        return VCA_ERR_CUDA;
    }
    return VCA_OK;
}

// the w = 4 family runs small_block_kernel (thread per block) unless the warp-generic
// kernel is forced for every family
inline bool small_path(const vca_ctx *c)
{
#ifdef VCA_FORCE_GENERIC
    (void)c;
    return false;
#else
    return c->path == VCA_PATH_WARP_GENERIC && c->geo[0].n == 4 && c->geo[1].n == 4 && !c->lowpass;
#endif
}

#define VCA_CK(ctx, call)                                    \
    do {                                                     \
        cudaError_t e_ = (call);                             \
        if (e_ != cudaSuccess) return fail_cuda((ctx), e_);  \
    } while (0)

// R-1: T_n[k][x] = round(64 sqrt(2) c_k cos(pi (2x+1) k / 2n)), c_0 = 1/sqrt(2).
void make_basis(int n, int8_t *T)
{
    const double pi = 3.14159265358979323846;
    for (int k = 0; k < n; ++k)
        for (int x = 0; x < n; ++x) {
            const double ck = k == 0 ? std::sqrt(0.5) : 1.0;
            const double v = 64.0 * std::sqrt(2.0) * ck * std::cos(pi * (2 * x + 1) * k / (2.0 * n));
            T[k * n + x] = (int8_t)std::lround(v);
        }
}

// R-2, R-3: W_n(i,j) = exp(|(ij/n^2)^2 - 1|) / (4096 n); 0 at DC.
void make_weights(int n, double *W)
{
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double r = (double)(i * j) / (double)(n * n);
            W[i * n + j] = (i == 0 && j == 0) ? 0.0 : std::exp(std::fabs(r * r - 1.0)) / (4096.0 * n);
        }
}

int resolve_block(int height, int block_size)
{
    if (block_size == 0) return height >= 2160 ? 32 : (height >= 1080 ? 16 : 8);
    return block_size;
}

void set_geo(PlaneDesc &g, int pw, int ph, int w, int lowpass)
{
    g.base = nullptr;
    g.pitch = g.fstride = 0;
    g.width = pw;
    g.height = ph;
    g.w = w;
    g.n = lowpass ? w / 2 : w;
    g.cols = (pw + w - 1) / w;
    g.rows = (ph + w - 1) / w;
    g.count = (int64_t)g.cols * g.rows;
}

int elem_bytes(const vca_ctx *c) { return c->bd == 8 ? 1 : 2; }

int check_planes(const vca_ctx *ctx, const void *const planes[3], const int64_t pitch[3],
                 const int64_t fstride[3], int n_frames)
{
    if (!planes || !pitch || !fstride) return VCA_ERR_INVALID_ARG;
    for (int p = 0; p < 3; ++p) {
        if (!planes[p]) return VCA_ERR_INVALID_ARG;
        const int64_t row_bytes = (int64_t)ctx->geo[p].width * elem_bytes(ctx);
        if (pitch[p] < row_bytes) return VCA_ERR_INVALID_ARG;
        if (n_frames > 1 && fstride[p] < pitch[p] * ctx->geo[p].height) return VCA_ERR_INVALID_ARG;
        if (((uintptr_t)planes[p] & 15) || (pitch[p] & 15) || (fstride[p] & 15)) return VCA_ERR_ALIGNMENT;
    }
    return VCA_OK;
}

size_t scratch_bytes(const vca_ctx *c, int F)
{
    return sizeof(double) * ((size_t)F * (size_t)c->geo[0].count + (size_t)F * 3 * (size_t)c->P * 2);
}

EventTriple take_events(vca_ctx *ctx, cudaError_t *err)
{
    EventTriple t{};
    *err = cudaSuccess;
    if (!ctx->pool.empty()) {
        t = ctx->pool.back();
        ctx->pool.pop_back();
        return t;
    }
    for (int i = 0; i < 3; ++i) {
        *err = cudaEventCreate(&t.e[i]);
        if (*err != cudaSuccess) return t;
    }
    return t;
}

Planes3 make_planes(const vca_ctx *ctx, const void *const planes[3], const int64_t pitch[3], const int64_t fstride[3])
{
    Planes3 pl;
    for (int p = 0; p < 3; ++p) {
        pl.p[p] = ctx->geo[p];
        pl.p[p].base = static_cast<const uint8_t *>(planes[p]);
        pl.p[p].pitch = pitch[p];
        pl.p[p].fstride = fstride[p];
    }
    return pl;
}

// The argument checks launch_analysis makes before enqueuing anything (tensor maps encodable,
// work counts in range), without launching: VCA_OK or VCA_ERR_INVALID_ARG.
int validate_launch(const vca_ctx *ctx, const void *const planes[3], const int64_t pitch[3], const int64_t fstride[3],
                    int n_frames)
{
    if (ctx->path == VCA_PATH_FUSED_MMA)
        return fused_check(make_planes(ctx, planes, pitch, fstride), n_frames, ctx->bd, ctx->lowpass) ? VCA_OK
                                                                                                       : VCA_ERR_INVALID_ARG;
    const int64_t per_frame = ctx->geo[0].count + ctx->geo[1].count + ctx->geo[2].count;
    return per_frame > 0x7fffffff ? VCA_ERR_INVALID_ARG : VCA_OK;
}

// Enqueue one analysis of n_frames frames (validated) on `st`.
int launch_analysis(vca_ctx *ctx, const void *const planes[3], const int64_t pitch[3], const int64_t fstride[3],
                    int n_frames, int n_halo, void *scratch, vca_features *out, cudaStream_t st,
                    const DumpPtrs *dump)
{
    const Planes3 pl = make_planes(ctx, planes, pitch, fstride);
    Scratch s;
    s.HY = static_cast<double *>(scratch);
    s.partial = s.HY + (size_t)n_frames * (size_t)ctx->geo[0].count;
    s.P = ctx->P;
    for (int p = 0; p < 3; ++p) s.Pp[p] = ctx->Pp[p];
    DumpPtrs nodump;
    memset(&nodump, 0, sizeof(nodump));
    const DumpPtrs &dp = dump ? *dump : nodump;

    EventTriple ev{};
    const bool prof = ctx->prof && !dump;
    if (prof) {
        cudaError_t e;
        ev = take_events(ctx, &e);
        VCA_CK(ctx, e);
        VCA_CK(ctx, cudaEventRecord(ev.e[0], st));
    }
    if (ctx->path == VCA_PATH_FUSED_MMA) {
        const int rc = launch_fused(pl, n_frames, ctx->bd, ctx->lowpass, ctx->d_T, ctx->d_W, s, dp, ctx->sm_count, st,
                                    ctx->d_ticket, &ctx->ticket_base);
        if (rc == -2) return VCA_ERR_INVALID_ARG;  // tensor map not encodable for these strides
    } else {
        const int64_t tasks = (int64_t)n_frames * (ctx->geo[0].count + ctx->geo[1].count + ctx->geo[2].count);
        int64_t blocks = (tasks + kGenericWarps - 1) / kGenericWarps;
        const int64_t cap = (int64_t)ctx->sm_count * 16;
        if (blocks > cap) blocks = cap;
#ifndef VCA_FORCE_GENERIC
        if (small_path(ctx)) {  // w = 4: thread per block, warp per 32-block chunk
            const int64_t per_frame = ctx->geo[0].count + ctx->geo[1].count + ctx->geo[2].count;
            if (per_frame > 0x7fffffff) return VCA_ERR_INVALID_ARG;
            const int64_t chunks = (int64_t)n_frames * (ctx->Pp[0] + ctx->Pp[1] + ctx->Pp[2]);
            int64_t tb = (chunks + 7) / 8;  // 8 warps per 256-thread CTA
            const int64_t tcap = (int64_t)ctx->sm_count * 8;
            if (tb > tcap) tb = tcap;
            const bool dmp = dp.on != 0;
            if (ctx->bd == 8) {
                if (dmp)
                    small_block_kernel<8, true><<<(unsigned)tb, 256, 0, st>>>(pl, n_frames, ctx->d_T, ctx->d_W, s, dp);
                else
                    small_block_kernel<8, false><<<(unsigned)tb, 256, 0, st>>>(pl, n_frames, ctx->d_T, ctx->d_W, s, dp);
            } else {
                if (dmp)
                    small_block_kernel<10, true><<<(unsigned)tb, 256, 0, st>>>(pl, n_frames, ctx->d_T, ctx->d_W, s, dp);
                else
                    small_block_kernel<10, false><<<(unsigned)tb, 256, 0, st>>>(pl, n_frames, ctx->d_T, ctx->d_W, s, dp);
            }
        } else
#endif
        if (ctx->bd == 8)
            generic_block_kernel<8><<<(unsigned)blocks, 32 * kGenericWarps, 0, st>>>(pl, n_frames, ctx->lowpass,
                                                                                    ctx->d_T, ctx->d_W, s, dp);
        else
            generic_block_kernel<10><<<(unsigned)blocks, 32 * kGenericWarps, 0, st>>>(pl, n_frames, ctx->lowpass,
                                                                                     ctx->d_T, ctx->d_W, s, dp);
    }
    VCA_CK(ctx, cudaGetLastError());
    ctx->launches += 1;
    if (!out) return VCA_OK;  // vca_debug_dump: no records, no state change
    if (prof) VCA_CK(ctx, cudaEventRecord(ev.e[1], st));

    FinalizeArgs fa;
    fa.s = s;
    fa.n_frames = n_frames;
    fa.n_halo = n_halo;
    for (int p = 0; p < 3; ++p) {
        fa.count[p] = ctx->geo[p].count;
        fa.n[p] = ctx->geo[p].n;
    }
    const size_t CY = (size_t)ctx->geo[0].count;
    fa.prevHY = (n_halo == 0 && ctx->prev_valid) ? ctx->d_prevHY + ctx->cur_prev * CY : nullptr;
    fa.saveHY = ctx->d_prevHY + (1 - ctx->cur_prev) * CY;
    fa.first_poc = ctx->next_poc;
    fa.out = out;
    // several consecutive frames per CTA (each H_Y read once) while the grid still covers the SMs
    fa.frames_per_cta = 1;
    if (CY <= (size_t)kFinalizeThreads * kHYRegs)
        for (int k = VCA_FIN_FRAMES; k > 1; k >>= 1)
            if (n_frames >= k * ctx->sm_count) {
                fa.frames_per_cta = k;
                break;
            }
    const int fin_grid = (n_frames + fa.frames_per_cta - 1) / fa.frames_per_cta;
    if (fa.frames_per_cta > 1)
        finalize_kernel<true><<<fin_grid, kFinalizeThreads, 0, st>>>(fa);
    else
        finalize_kernel<false><<<fin_grid, kFinalizeThreads, 0, st>>>(fa);
    VCA_CK(ctx, cudaGetLastError());
    ctx->launches += 1;
    if (prof) {
        VCA_CK(ctx, cudaEventRecord(ev.e[2], st));
        ctx->pending.push_back(ev);
    }
    // the finalize kernel wrote the last frame's H_Y into the other buffer (R-7)
    ctx->cur_prev = 1 - ctx->cur_prev;
    ctx->prev_valid = true;
    ctx->next_poc += n_frames - n_halo;
    return VCA_OK;
}

}  // namespace

extern "C" {

const char *vca_version(void) { return "vca-b200 0.1"; }

const char *vca_status_string(int status)
{
    switch (status) {
    case VCA_OK: return "ok";
    case VCA_ERR_INVALID_ARG: return "invalid argument";
    case VCA_ERR_UNSUPPORTED_BLOCK_SIZE: return "unsupported block size";
    case VCA_ERR_UNSUPPORTED_BIT_DEPTH: return "unsupported bit depth";
    case VCA_ERR_UNSUPPORTED_CHROMA: return "unsupported chroma format";
    case VCA_ERR_GEOMETRY: return "invalid geometry";
    case VCA_ERR_ALIGNMENT: return "misaligned plane, pitch or frame stride (16 bytes required)";
    case VCA_ERR_CUDA: return "CUDA error (context poisoned)";
    case VCA_ERR_OOM: return "out of device memory";
    case VCA_ERR_SCRATCH: return "scratch buffer too small";
    case VCA_IO_EOF: return "end of stream";
    case VCA_ERR_IO: return "I/O error (open, read or write)";
    case VCA_ERR_MALFORMED_MAGIC: return "not a Y4M stream (missing YUV4MPEG2 magic)";
    case VCA_ERR_MALFORMED_HEADER: return "malformed Y4M header or stream geometry";
    case VCA_ERR_TRUNCATED_FRAME: return "truncated frame";
    case VCA_ERR_MALFORMED_FRAME_MARKER: return "malformed Y4M FRAME marker";
    case VCA_ERR_INTERLACED: return "interlaced Y4M stream (progressive only)";
    default: return "unknown status";
    }
}

int vca_create(int width, int height, int bit_depth, int chroma_format, int block_size, int lowpass, vca_ctx **out)
{
    if (!out) return VCA_ERR_INVALID_ARG;
    if (bit_depth != 8 && bit_depth != 10) return VCA_ERR_UNSUPPORTED_BIT_DEPTH;
    if (chroma_format != VCA_CHROMA_420) return VCA_ERR_UNSUPPORTED_CHROMA;
    if (width < 2 || height < 2 || (width & 1) || (height & 1) || width > (1 << 16) || height > (1 << 16))
        return VCA_ERR_GEOMETRY;
    if (lowpass != 0 && lowpass != 1) return VCA_ERR_INVALID_ARG;
    if (!(block_size == 0 || block_size == 4 || block_size == 8 || block_size == 16 || block_size == 32))
        return VCA_ERR_UNSUPPORTED_BLOCK_SIZE;
    const int w = resolve_block(height, block_size);
    const int wc = w / 2 < 4 ? 4 : w / 2;
    if (lowpass && wc < 8) return VCA_ERR_UNSUPPORTED_BLOCK_SIZE;

    vca_ctx *c = new (std::nothrow) vca_ctx();
    if (!c) return VCA_ERR_OOM;
    c->width = width;
    c->height = height;
    c->bd = bit_depth;
    c->lowpass = lowpass;
    set_geo(c->geo[0], width, height, w, lowpass);
    set_geo(c->geo[1], width / 2, height / 2, wc, lowpass);
    set_geo(c->geo[2], width / 2, height / 2, wc, lowpass);
    c->path = fused_supported(w, lowpass, c->geo[0].cols == c->geo[1].cols && c->geo[0].rows == c->geo[1].rows)
                  ? VCA_PATH_FUSED_MMA
                  : VCA_PATH_WARP_GENERIC;
    if (c->path == VCA_PATH_FUSED_MMA) {
        const int pr = fused_partials_per_row();
        for (int p = 0; p < 3; ++p) c->Pp[p] = c->geo[p].rows * pr;
    } else if (small_path(c)) {
        for (int p = 0; p < 3; ++p)  // one partial per chunk of 32 VCA_W4_B blocks
            c->Pp[p] = (int)((c->geo[p].count + 32 * VCA_W4_B - 1) / (32 * VCA_W4_B));
    } else {
        for (int p = 0; p < 3; ++p) c->Pp[p] = (int)c->geo[p].count;
    }
    c->P = c->Pp[0] > c->Pp[1] ? c->Pp[0] : c->Pp[1];

    int8_t hT[kTableElems];
    double hW[kTableElems];
    for (int n = 4; n <= 32; n *= 2) {
        make_basis(n, hT + table_offset(n));
        make_weights(n, hW + table_offset(n));
    }
    cudaError_t e = cudaGetDevice(&c->device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_T, sizeof(hT));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_W, sizeof(hW));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_prevHY, 2 * sizeof(double) * (size_t)c->geo[0].count);
    if (e == cudaSuccess) e = cudaMalloc(&c->d_ticket, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(c->d_ticket, 0, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemcpy(c->d_T, hT, sizeof(hT), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(c->d_W, hW, sizeof(hW), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && c->path == VCA_PATH_FUSED_MMA) e = fused_prepare(c->bd, c->lowpass, w);
    if (e != cudaSuccess) {
        const int rc = e == cudaErrorMemoryAllocation ? VCA_ERR_OOM : VCA_ERR_CUDA;
        vca_destroy(c);
        cudaGetLastError();
        return rc;
    }
    *out = c;
    return VCA_OK;
}

int vca_get_info(const vca_ctx *ctx, vca_info *info)
{
    if (!ctx || !info) return VCA_ERR_INVALID_ARG;
    info->width = ctx->width;
    info->height = ctx->height;
    info->bit_depth = ctx->bd;
    info->lowpass = ctx->lowpass;
    for (int p = 0; p < 3; ++p) {
        info->block[p] = ctx->geo[p].w;
        info->n[p] = ctx->geo[p].n;
        info->cols[p] = ctx->geo[p].cols;
        info->rows[p] = ctx->geo[p].rows;
        info->count[p] = ctx->geo[p].count;
    }
    info->path = ctx->path;
    return VCA_OK;
}

size_t vca_scratch_bytes(const vca_ctx *ctx, int max_frames)
{
    if (!ctx || max_frames < 1) return 0;
    return scratch_bytes(ctx, max_frames);
}

int vca_analyze(vca_ctx *ctx, const void *const planes[3], const int64_t pitch_bytes[3],
                const int64_t frame_stride_bytes[3], int n_frames, int n_halo, void *scratch, size_t scratch_bytes_,
                vca_features *out_dev, void *stream)
{
    if (!ctx) return VCA_ERR_INVALID_ARG;
    if (ctx->poisoned) return VCA_ERR_CUDA;
    if (n_halo < 0 || n_halo > 1 || n_frames < 1 + n_halo || !out_dev || !scratch) return VCA_ERR_INVALID_ARG;
    int rc = check_planes(ctx, planes, pitch_bytes, frame_stride_bytes, n_frames);
    if (rc) return rc;
    if (((uintptr_t)scratch & 7) || scratch_bytes_ < scratch_bytes(ctx, n_frames)) return VCA_ERR_SCRATCH;
    return launch_analysis(ctx, planes, pitch_bytes, frame_stride_bytes, n_frames, n_halo, scratch, out_dev,
                           static_cast<cudaStream_t>(stream), nullptr);
}

int vca_analyze_host(vca_ctx *ctx, const void *const host_planes[3], const int64_t pitch_bytes[3],
                     const int64_t frame_stride_bytes[3], int n_frames, int n_halo, int chunk_frames,
                     vca_features *out_host, void *stream)
{
    if (!ctx) return VCA_ERR_INVALID_ARG;
    if (ctx->poisoned) return VCA_ERR_CUDA;
    if (n_halo < 0 || n_halo > 1 || n_frames < 1 + n_halo || !out_host) return VCA_ERR_INVALID_ARG;
    int rc = check_planes(ctx, host_planes, pitch_bytes, frame_stride_bytes, n_frames);
    if (rc) return rc;
    if (chunk_frames <= 0) chunk_frames = 8;
    if (chunk_frames > n_frames) chunk_frames = n_frames;
    cudaStream_t user = static_cast<cudaStream_t>(stream);

    // device staging of one chunk, plane-major: [Y frames][U frames][V frames], rows of
    // round16(row bytes), so a chunk of host frames stored back to back is one 2-D copy per plane
    int64_t dpitch[3], dfs[3], off[3];
    size_t frame_bytes = 0;
    for (int p = 0; p < 3; ++p) {
        dpitch[p] = (((int64_t)ctx->geo[p].width * elem_bytes(ctx)) + 15) & ~(int64_t)15;
        dfs[p] = dpitch[p] * ctx->geo[p].height;
        off[p] = (int64_t)frame_bytes * chunk_frames;
        frame_bytes += (size_t)dfs[p];
    }
    // (re)allocate context-owned staging when the chunk grows
    const size_t need = frame_bytes * (size_t)chunk_frames;
    if (need > ctx->stage_bytes || chunk_frames > ctx->stage_frames) {
        // any failure leaves no staging at all (sizes 0, pointers NULL), so a later call
        // reallocates instead of launching on a partial set of buffers
        auto drop = [ctx]() {
            for (int b = 0; b < 2; ++b) {
                if (ctx->stage[b]) cudaFree(ctx->stage[b]);
                ctx->stage[b] = nullptr;
            }
            if (ctx->h_scratch) cudaFree(ctx->h_scratch);
            ctx->h_scratch = nullptr;
            ctx->stage_bytes = 0;
            ctx->stage_frames = 0;
            ctx->h_scratch_bytes = 0;
        };
        drop();
        cudaError_t e = cudaSuccess;
        for (int b = 0; b < 2 && e == cudaSuccess; ++b) e = cudaMalloc(&ctx->stage[b], need);
        const size_t hsb = scratch_bytes(ctx, chunk_frames);
        if (e == cudaSuccess) e = cudaMalloc(&ctx->h_scratch, 2 * hsb);
        if (e != cudaSuccess) {
            cudaGetLastError();
            drop();
            return e == cudaErrorMemoryAllocation ? VCA_ERR_OOM : fail_cuda(ctx, e);
        }
        ctx->h_scratch_bytes = hsb;
        ctx->stage_bytes = need;
        ctx->stage_frames = chunk_frames;
    }
    if ((size_t)n_frames > ctx->d_rec_n) {
        if (ctx->d_rec) cudaFree(ctx->d_rec);
        ctx->d_rec = nullptr;
        cudaError_t e = cudaMalloc(&ctx->d_rec, sizeof(vca_features) * (size_t)n_frames);
        if (e != cudaSuccess) {
            cudaGetLastError();
            ctx->d_rec_n = 0;
            return e == cudaErrorMemoryAllocation ? VCA_ERR_OOM : fail_cuda(ctx, e);
        }
        ctx->d_rec_n = (size_t)n_frames;
    }
    if (!ctx->s_copy) {
        VCA_CK(ctx, cudaStreamCreateWithFlags(&ctx->s_copy, cudaStreamNonBlocking));
        VCA_CK(ctx, cudaStreamCreateWithFlags(&ctx->s_comp, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            VCA_CK(ctx, cudaEventCreateWithFlags(&ctx->ev_copied[b], cudaEventDisableTiming));
            VCA_CK(ctx, cudaEventCreateWithFlags(&ctx->ev_done[b], cudaEventDisableTiming));
        }
    }
    // order the internal streams after prior work on the user's stream
    cudaEvent_t start_ev = ctx->ev_done[0];
    VCA_CK(ctx, cudaEventRecord(start_ev, user));
    VCA_CK(ctx, cudaStreamWaitEvent(ctx->s_copy, start_ev, 0));
    VCA_CK(ctx, cudaStreamWaitEvent(ctx->s_comp, start_ev, 0));

    // validate every chunk geometry (full chunks and the last, shorter one) before anything is
    // enqueued, so an argument error leaves the context unchanged (vca.h)
    {
        const void *dpl[3] = {ctx->stage[0] + off[0], ctx->stage[0] + off[1], ctx->stage[0] + off[2]};
        const int last = n_frames % chunk_frames;
        rc = validate_launch(ctx, dpl, dpitch, dfs, chunk_frames);
        if (rc == VCA_OK && last) rc = validate_launch(ctx, dpl, dpitch, dfs, last);
        if (rc) return rc;
    }
    int emitted = 0;
    int k = 0;
    bool used[2] = {false, false};
    for (int f0 = 0; f0 < n_frames; f0 += chunk_frames, ++k) {
        const int m = (n_frames - f0) < chunk_frames ? (n_frames - f0) : chunk_frames;
        const int b = k & 1;
        if (used[b]) VCA_CK(ctx, cudaStreamWaitEvent(ctx->s_copy, ctx->ev_done[b], 0));
        uint8_t *dst = ctx->stage[b];
        for (int p = 0; p < 3; ++p) {
            const uint8_t *src = static_cast<const uint8_t *>(host_planes[p]) + (int64_t)f0 * frame_stride_bytes[p];
            const size_t wbytes = (size_t)ctx->geo[p].width * elem_bytes(ctx);
            const int h = ctx->geo[p].height;
            if (frame_stride_bytes[p] == pitch_bytes[p] * h)  // frames back to back: one copy of m*h rows
                VCA_CK(ctx, cudaMemcpy2DAsync(dst + off[p], (size_t)dpitch[p], src, (size_t)pitch_bytes[p], wbytes,
                                              (size_t)h * m, cudaMemcpyHostToDevice, ctx->s_copy));
            else
                for (int t = 0; t < m; ++t)
                    VCA_CK(ctx, cudaMemcpy2DAsync(dst + off[p] + (size_t)t * dfs[p], (size_t)dpitch[p],
                                                  src + (int64_t)t * frame_stride_bytes[p], (size_t)pitch_bytes[p],
                                                  wbytes, (size_t)h, cudaMemcpyHostToDevice, ctx->s_copy));
        }
        VCA_CK(ctx, cudaEventRecord(ctx->ev_copied[b], ctx->s_copy));
        VCA_CK(ctx, cudaStreamWaitEvent(ctx->s_comp, ctx->ev_copied[b], 0));
        const void *dpl[3] = {dst + off[0], dst + off[1], dst + off[2]};
        int64_t dfstride[3] = {dfs[0], dfs[1], dfs[2]};
        const int halo = (f0 == 0) ? n_halo : 0;
        void *scr = static_cast<uint8_t *>(ctx->h_scratch) + (size_t)b * ctx->h_scratch_bytes;
        if (m - halo > 0 || halo) {
            rc = launch_analysis(ctx, dpl, dpitch, dfstride, m, halo, scr, ctx->d_rec + emitted, ctx->s_comp, nullptr);
            if (rc) {
                // unreachable for argument errors (every chunk geometry was validated above);
                // a CUDA error has poisoned the context already
                ctx->poisoned = true;
                return rc == VCA_ERR_CUDA ? rc : VCA_ERR_CUDA;
            }
        }
        emitted += m - halo;
        VCA_CK(ctx, cudaEventRecord(ctx->ev_done[b], ctx->s_comp));
        used[b] = true;
    }
    VCA_CK(ctx, cudaMemcpyAsync(out_host, ctx->d_rec, sizeof(vca_features) * (size_t)emitted, cudaMemcpyDeviceToHost,
                                ctx->s_comp));
    VCA_CK(ctx, cudaStreamSynchronize(ctx->s_comp));
    return VCA_OK;
}

int vca_reset(vca_ctx *ctx, int64_t next_poc)
{
    if (!ctx) return VCA_ERR_INVALID_ARG;
    if (ctx->poisoned) return VCA_ERR_CUDA;
    ctx->prev_valid = false;
    ctx->next_poc = next_poc;
    return VCA_OK;
}

int vca_profile_enable(vca_ctx *ctx, int enable)
{
    if (!ctx) return VCA_ERR_INVALID_ARG;
    ctx->prof = enable != 0;
    return VCA_OK;
}

int vca_profile_read(vca_ctx *ctx, double *block_kernel_ms, double *finalize_ms, int64_t *launches)
{
    if (!ctx) return VCA_ERR_INVALID_ARG;
    if (ctx->poisoned) return VCA_ERR_CUDA;
    for (auto &t : ctx->pending) {
        VCA_CK(ctx, cudaEventSynchronize(t.e[2]));
        float a = 0, b = 0;
        VCA_CK(ctx, cudaEventElapsedTime(&a, t.e[0], t.e[1]));
        VCA_CK(ctx, cudaEventElapsedTime(&b, t.e[1], t.e[2]));
        ctx->acc_block_ms += a;
        ctx->acc_fin_ms += b;
        ctx->pool.push_back(t);
    }
    ctx->pending.clear();
    if (block_kernel_ms) *block_kernel_ms = ctx->acc_block_ms;
    if (finalize_ms) *finalize_ms = ctx->acc_fin_ms;
    if (launches) *launches = ctx->launches;
    ctx->acc_block_ms = ctx->acc_fin_ms = 0;
    ctx->launches = 0;
    return VCA_OK;
}

int vca_debug_dump(vca_ctx *ctx, const void *const planes[3], const int64_t pitch_bytes[3],
                   int32_t *const coeffs[3], int64_t *const sumx[3], double *const H[3], double *const L[3])
{
    if (!ctx || !coeffs || !sumx || !H || !L) return VCA_ERR_INVALID_ARG;
    if (ctx->poisoned) return VCA_ERR_CUDA;
    int64_t fs[3] = {0, 0, 0};
    for (int p = 0; p < 3; ++p) fs[p] = pitch_bytes ? pitch_bytes[p] * ctx->geo[p].height : 0;
    int rc = check_planes(ctx, planes, pitch_bytes, fs, 1);
    if (rc) return rc;
    DumpPtrs dp;
    memset(&dp, 0, sizeof(dp));
    dp.on = 1;
    void *scratch = nullptr;
    rc = VCA_OK;
    cudaError_t e = cudaMalloc(&scratch, scratch_bytes(ctx, 1));
    for (int p = 0; p < 3 && e == cudaSuccess; ++p) {
        if (!coeffs[p]) continue;
        const int64_t C = ctx->geo[p].count, n = ctx->geo[p].n;
        e = cudaMalloc(&dp.coeffs[p], sizeof(int32_t) * C * n * n);
        if (e == cudaSuccess) e = cudaMalloc(&dp.sumx[p], sizeof(int64_t) * C);
        if (e == cudaSuccess) e = cudaMalloc(&dp.H[p], sizeof(double) * C);
        if (e == cudaSuccess) e = cudaMalloc(&dp.L[p], sizeof(double) * C);
    }
    if (e == cudaSuccess) {
        rc = launch_analysis(ctx, planes, pitch_bytes, fs, 1, 0, scratch, nullptr, nullptr, &dp);
        if (rc == VCA_OK) e = cudaDeviceSynchronize();
    }
    for (int p = 0; p < 3 && e == cudaSuccess && rc == VCA_OK; ++p) {
        if (!coeffs[p]) continue;
        const int64_t C = ctx->geo[p].count, n = ctx->geo[p].n;
        e = cudaMemcpy(coeffs[p], dp.coeffs[p], sizeof(int32_t) * C * n * n, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && sumx[p]) e = cudaMemcpy(sumx[p], dp.sumx[p], sizeof(int64_t) * C, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && H[p]) e = cudaMemcpy(H[p], dp.H[p], sizeof(double) * C, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && L[p]) e = cudaMemcpy(L[p], dp.L[p], sizeof(double) * C, cudaMemcpyDeviceToHost);
    }
    for (int p = 0; p < 3; ++p) {
        cudaFree(dp.coeffs[p]);
        cudaFree(dp.sumx[p]);
        cudaFree(dp.H[p]);
        cudaFree(dp.L[p]);
    }
    cudaFree(scratch);
    if (rc) return rc;
    return fail_cuda(ctx, e);
}

int vca_debug_analyze(vca_ctx *ctx, const void *const planes[3], const int64_t pitch_bytes[3],
                      const int64_t frame_stride_bytes[3], int n_frames, int n_halo, void *scratch,
                      size_t scratch_bytes_, vca_features *out_dev, int64_t *const chk_dev[3],
                      int64_t *const sumx_dev[3], double *const H_dev[3], void *stream)
{
    if (!ctx) return VCA_ERR_INVALID_ARG;
    if (ctx->poisoned) return VCA_ERR_CUDA;
    if (n_halo < 0 || n_halo > 1 || n_frames < 1 + n_halo || !out_dev || !scratch) return VCA_ERR_INVALID_ARG;
    int rc = check_planes(ctx, planes, pitch_bytes, frame_stride_bytes, n_frames);
    if (rc) return rc;
    if (((uintptr_t)scratch & 7) || scratch_bytes_ < scratch_bytes(ctx, n_frames)) return VCA_ERR_SCRATCH;
    rc = validate_launch(ctx, planes, pitch_bytes, frame_stride_bytes, n_frames);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DumpPtrs dp;
    memset(&dp, 0, sizeof(dp));
    dp.on = 1;
    for (int p = 0; p < 3; ++p) {
        dp.chk[p] = chk_dev ? reinterpret_cast<unsigned long long *>(chk_dev[p]) : nullptr;
        dp.sumx[p] = sumx_dev ? sumx_dev[p] : nullptr;
        dp.H[p] = H_dev ? H_dev[p] : nullptr;
        if (dp.chk[p])
            VCA_CK(ctx, cudaMemsetAsync(dp.chk[p], 0, sizeof(int64_t) * (size_t)n_frames * (size_t)ctx->geo[p].count, st));
    }
    return launch_analysis(ctx, planes, pitch_bytes, frame_stride_bytes, n_frames, n_halo, scratch, out_dev, st, &dp);
}

#ifdef VCA_TIMES
// diagnostic build only: copies, for n consumer groups of the last fused launch, the start and
// end globaltimer stamps (ns) and the SM id, as three arrays of n
int vca_debug_group_times(unsigned long long *host, int n)
{
    if (!host || n < 0 || n > 4096) return VCA_ERR_INVALID_ARG;
    if (cudaMemcpyFromSymbol(host, vca_group_t, sizeof(unsigned long long) * n, 0) != cudaSuccess) return VCA_ERR_CUDA;
    if (cudaMemcpyFromSymbol(host + n, vca_group_t, sizeof(unsigned long long) * n,
                             sizeof(unsigned long long) * 4096) != cudaSuccess)
        return VCA_ERR_CUDA;
    if (cudaMemcpyFromSymbol(host + 2 * n, vca_group_t, sizeof(unsigned long long) * n,
                             sizeof(unsigned long long) * 8192) != cudaSuccess)
        return VCA_ERR_CUDA;
    return VCA_OK;
}
#endif

int vca_debug_mutate(int plane, int64_t block, int pos, int which)
{
#ifdef VCA_MUTATE
    MutSpec m;
    m.plane = plane;
    m.block = block;
    m.pos = pos;
    m.which = which;
    return cudaMemcpyToSymbol(vca_mut, &m, sizeof(m)) == cudaSuccess ? VCA_OK : VCA_ERR_CUDA;
#else
    (void)plane;
    (void)block;
    (void)pos;
    (void)which;
    return VCA_ERR_INVALID_ARG;  // not a VCA_MUTATE build
#endif
}

void vca_destroy(vca_ctx *ctx)
{
    if (!ctx) return;
    cudaFree(ctx->d_T);
    cudaFree(ctx->d_W);
    cudaFree(ctx->d_prevHY);
    cudaFree(ctx->d_ticket);
    for (int b = 0; b < 2; ++b) cudaFree(ctx->stage[b]);
    cudaFree(ctx->h_scratch);
    cudaFree(ctx->d_rec);
    if (ctx->s_copy) cudaStreamDestroy(ctx->s_copy);
    if (ctx->s_comp) cudaStreamDestroy(ctx->s_comp);
    for (int b = 0; b < 2; ++b) {
        if (ctx->ev_copied[b]) cudaEventDestroy(ctx->ev_copied[b]);
        if (ctx->ev_done[b]) cudaEventDestroy(ctx->ev_done[b]);
    }
    for (auto &t : ctx->pool)
        for (int i = 0; i < 3; ++i) cudaEventDestroy(t.e[i]);
    for (auto &t : ctx->pending)
        for (int i = 0; i < 3; ++i) cudaEventDestroy(t.e[i]);
    delete ctx;
}

}  // extern "C"
