/*
 * vca_io.h -- C ABI of libvca's host-side ingest, streaming driver and CSV
 * writer: Y4M / raw-YUV frame sources read into
 * pinned host buffers by a reader thread while the GPU analyses the previous
 * batch, and the per-frame features CSV.
 *
 * Citations: S:n = SPEC.md line n (the ingest module S:24-93, stats S:402-469,
 * cli S:471-508), R-k = DESIGN.md reading k (R-13..R-16 cover the ingest).
 * This is plumbing around the hot path, not part of it: the paper does not say
 * how VCA ingests content, Y4M + raw YUV is SPEC's choice.
 *
 * Conventions: as vca.h -- return VCA_OK (0), VCA_IO_EOF (1, readers only) or
 * a negative code; nothing is thrown across the ABI; the caller owns every
 * buffer passed in; a reader must not be used from two threads at once.
 * These calls are host-only (no CUDA) except vca_analyze_stream.
 */
#ifndef VCA_IO_H
#define VCA_IO_H

#include "vca.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
    VCA_IO_EOF = 1,                     /* clean end of stream at a frame boundary          */
    VCA_ERR_IO = -10,                   /* file not found / read error / write error        */
    VCA_ERR_MALFORMED_MAGIC = -11,      /* Y4M stream does not start with "YUV4MPEG2 "      */
    VCA_ERR_MALFORMED_HEADER = -12,     /* unparsable or missing W/H/F token, bad geometry  */
    VCA_ERR_TRUNCATED_FRAME = -13,      /* Y4M frame payload shorter than one frame         */
    VCA_ERR_MALFORMED_FRAME_MARKER = -14,/* Y4M frame not introduced by "FRAME"             */
    VCA_ERR_INTERLACED = -15            /* Y4M I token other than progressive (Ip)          */
};
/* Header errors with no specific code above reuse vca.h's
 * VCA_ERR_UNSUPPORTED_CHROMA (mono, unknown C tag) and
 * VCA_ERR_UNSUPPORTED_BIT_DEPTH (C...p9, p12, ...). */

/* Warning bits (vca_reader_warnings). */
enum {
    VCA_WARN_TRAILING_BYTES = 1,  /* raw file size not a multiple of the frame size: partial frame discarded */
    VCA_WARN_X_TOKENS = 2         /* Y4M X (extension) tokens ignored                                      */
};

/* Stream geometry. chroma_format: VCA_CHROMA_420/422/444.
 * bytes_per_sample: 1 (8-bit) or 2 (10-bit, little-endian uint16 containers).
 * frame_bytes: payload bytes of one frame (luma + 2 chroma planes).
 * frame_count: number of whole frames if known from the file size, else -1
 * (pipes, Y4M with per-frame parameters). */
typedef struct {
    int width, height, bit_depth, chroma_format;
    int fps_num, fps_den;
    int bytes_per_sample;
    int chroma_width, chroma_height;
    int64_t frame_bytes;
    int64_t frame_count;
} vca_stream_info;

typedef struct vca_reader vca_reader;

/* Parse a Y4M stream header from bytes[0..len): "YUV4MPEG2" then
 * space-separated tokens W<int> H<int> F<num>:<den> I<p> A<n>:<d> C<tag>
 * X<...>, terminated by '\n'.  C tags: 420jpeg/420mpeg2/420paldv/420 -> 4:2:0
 * 8-bit, 422, 444, and the p10 forms -> 10-bit; absent C -> 420jpeg (the Y4M
 * default).  W, H and F are required (F num, den > 0); 4:2:0 needs even W and
 * H, 4:2:2 even W.  On success *header_len = bytes up to and including the
 * '\n'.  Errors: VCA_ERR_MALFORMED_MAGIC, VCA_ERR_MALFORMED_HEADER (also: no
 * '\n' within len), VCA_ERR_INTERLACED, VCA_ERR_UNSUPPORTED_CHROMA,
 * VCA_ERR_UNSUPPORTED_BIT_DEPTH.  *warnings (may be NULL) gets
 * VCA_WARN_X_TOKENS when X tokens were skipped. */
int vca_y4m_parse_header(const char *bytes, size_t len, vca_stream_info *info, size_t *header_len, int *warnings);

/* Open a Y4M file (path "-" = standard input) and parse its header.
 * *info receives the geometry; frame_count is derived from the file size
 * when the file is seekable (assuming bare "FRAME\n" markers), else -1.
 * VCA_ERR_IO if the file cannot be opened; header errors as above. */
int vca_y4m_open(const char *path, vca_reader **out, vca_stream_info *info);

/* Open a headerless planar raw YUV file (I420/I422/I444) with the
 * caller's geometry: width, height > 0 (even as the chroma format requires),
 * bit_depth 8 or 10.  frame_count = file size / frame_bytes; a trailing
 * partial frame is discarded and flagged VCA_WARN_TRAILING_BYTES (R-14).
 * Errors: VCA_ERR_IO, VCA_ERR_MALFORMED_HEADER (bad geometry),
 * VCA_ERR_UNSUPPORTED_BIT_DEPTH, VCA_ERR_UNSUPPORTED_CHROMA. */
int vca_raw_open(const char *path, int width, int height, int bit_depth, int chroma_format, vca_reader **out,
                 vca_stream_info *info);

/* Read up to max_frames frames in POC order into caller memory: frame t of
 * plane p goes to planes[p] + t * frame_stride_bytes[p], rows pitch_bytes[p]
 * apart (pitch >= row bytes).  Samples are copied raw (no range conversion,
 * S:59; 10-bit values > 1023 are clamped by the analyzer, R-10).
 * *n_read = frames delivered.  Returns VCA_OK if max_frames frames were read,
 * VCA_IO_EOF if the stream ended first (n_read may be > 0), or an error
 * (VCA_ERR_TRUNCATED_FRAME, VCA_ERR_MALFORMED_FRAME_MARKER, VCA_ERR_IO) after
 * delivering the *n_read whole frames before it.  Never reads past the
 * declared frame payload. */
int vca_reader_read(vca_reader *r, int max_frames, void *const planes[3], const int64_t pitch_bytes[3],
                    const int64_t frame_stride_bytes[3], int *n_read);

/* Frames delivered so far, and the warning bits collected so far. */
int64_t vca_reader_frames(const vca_reader *r);
int vca_reader_warnings(const vca_reader *r);
void vca_reader_close(vca_reader *r);

/* Stream a whole source through a context (the pipeline of S:359-364 with the
 * GPU as the worker): a reader thread fills one of two pinned host batches of
 * batch_frames frames while the context analyses the other with
 * vca_analyze_host (H2D chunks overlapped with the kernels), so file reading,
 * PCIe and the GPU overlap.  Records go to out_host in POC order, at most
 * capacity of them; the context's sequence state carries across calls, so a
 * caller may call again with more room: returns VCA_OK when capacity records
 * were produced and the source may have more, VCA_IO_EOF when the source is
 * exhausted, or an error (reader or analyzer code; *n_out records before it
 * are valid).  The source must be 4:2:0 with the context's geometry
 * (VCA_ERR_GEOMETRY otherwise).  *seconds (may be NULL) = wall time of the
 * analysis loop (reads + transfers + kernels).  batch_frames <= 0
 * selects 32. */
int vca_analyze_stream(vca_ctx *ctx, vca_reader *r, int batch_frames, vca_features *out_host, int64_t capacity,
                       int64_t *n_out, double *seconds);

/* Write the features CSV: header "POC,E_Y,h,L_Y,E_U,L_U,E_V,L_V",
 * one row per record "%lld,%.6f,...", '.' decimal separator independent of
 * the locale, LF newlines.  path "-" = standard output.  Returns
 * bytes written (>= 0) or VCA_ERR_IO. */
int64_t vca_write_csv(const char *path, const vca_features *rec, int64_t n);

/* Per-feature mean and max over n >= 1 records, summed in POC order
 * (S:429-436); mean[0..6], max[0..6] in CSV order E_Y, h, L_Y, E_U, L_U,
 * E_V, L_V.  VCA_ERR_INVALID_ARG for n < 1. */
int vca_summarize(const vca_features *rec, int64_t n, double mean[7], double max[7]);

#ifdef __cplusplus
}
#endif

#endif /* VCA_IO_H */
