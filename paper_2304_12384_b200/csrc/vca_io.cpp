// vca_io.cpp -- host-side ingest (Y4M / raw YUV), the streaming driver that
// overlaps file reads with the GPU, and the features CSV writer (include/vca_io.h;
// SURVEY.md §8(f) NEXT-3; SPEC.md ingest S:24-93, stats S:402-469, cli S:471-508).
// Plumbing around the hot path: no feature arithmetic lives here.
#include <cuda_runtime.h>
#include <locale.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unistd.h>
#include <algorithm>
#include <atomic>

#include "../../include/vca_io.h"

struct vca_reader {
    FILE *f = nullptr;
    bool own = false;  // close f on vca_reader_close (not stdin)
    bool y4m = false;
    vca_stream_info info{};
    int warnings = 0;
    int64_t frames = 0;
    bool done = false;
    // positional mode (regular files of fixed-size frame records): frame t's record starts
    // at data_off + t * rec_bytes and batches are read by several threads with pread
    int64_t data_off = -1, rec_bytes = 0, data_off_saved = 0;
};

namespace {

int chroma_dims(int chroma, int w, int h, int *cw, int *ch)
{
    switch (chroma) {
    case VCA_CHROMA_420:
        if ((w & 1) || (h & 1)) return VCA_ERR_MALFORMED_HEADER;
        *cw = w / 2;
        *ch = h / 2;
        return VCA_OK;
    case VCA_CHROMA_422:
        if (w & 1) return VCA_ERR_MALFORMED_HEADER;
        *cw = w / 2;
        *ch = h;
        return VCA_OK;
    case VCA_CHROMA_444:
        *cw = w;
        *ch = h;
        return VCA_OK;
    default:
        return VCA_ERR_UNSUPPORTED_CHROMA;
    }
}

int finish_info(vca_stream_info *in)
{
    if (in->width <= 0 || in->height <= 0 || in->width > (1 << 16) || in->height > (1 << 16))
        return VCA_ERR_MALFORMED_HEADER;
    if (in->bit_depth != 8 && in->bit_depth != 10) return VCA_ERR_UNSUPPORTED_BIT_DEPTH;
    int rc = chroma_dims(in->chroma_format, in->width, in->height, &in->chroma_width, &in->chroma_height);
    if (rc) return rc;
    in->bytes_per_sample = in->bit_depth == 8 ? 1 : 2;
    in->frame_bytes = ((int64_t)in->width * in->height + 2 * (int64_t)in->chroma_width * in->chroma_height) *
                      in->bytes_per_sample;
    return VCA_OK;
}

// strict decimal integer of a token body [s, e)
bool parse_int(const char *s, const char *e, long long *v)
{
    if (s >= e || e - s > 12) return false;
    long long x = 0;
    for (const char *p = s; p < e; ++p) {
        if (*p < '0' || *p > '9') return false;
        x = x * 10 + (*p - '0');
    }
    *v = x;
    return true;
}

bool parse_ratio(const char *s, const char *e, long long *a, long long *b)
{
    const char *c = (const char *)memchr(s, ':', (size_t)(e - s));
    return c && parse_int(s, c, a) && parse_int(c + 1, e, b);
}

int64_t file_size(FILE *f)
{
    long cur = ftell(f);
    if (cur < 0 || fseek(f, 0, SEEK_END) != 0) return -1;
    long end = ftell(f);
    fseek(f, cur, SEEK_SET);
    return end;
}

// read exactly n bytes; returns bytes read
size_t read_full(FILE *f, void *dst, size_t n)
{
    size_t got = 0;
    while (got < n) {
        size_t k = fread(static_cast<uint8_t *>(dst) + got, 1, n - got, f);
        if (k == 0) break;
        got += k;
    }
    return got;
}

// One frame's payload into plane rows; returns bytes read of this frame (== frame_bytes on success)
int64_t read_payload(vca_reader *r, void *const planes[3], const int64_t pitch[3], const int64_t fstride[3],
                     int t)
{
    const vca_stream_info &in = r->info;
    int64_t total = 0;
    for (int p = 0; p < 3; ++p) {
        const int w = p ? in.chroma_width : in.width, h = p ? in.chroma_height : in.height;
        const size_t rb = (size_t)w * in.bytes_per_sample;
        uint8_t *base = static_cast<uint8_t *>(planes[p]) + (int64_t)t * fstride[p];
        if ((size_t)pitch[p] == rb) {  // dense plane: one read
            const size_t k = read_full(r->f, base, rb * h);
            total += (int64_t)k;
            if (k < rb * h) return total;
        } else {
            for (int y = 0; y < h; ++y) {
                const size_t k = read_full(r->f, base + (int64_t)y * pitch[p], rb);
                total += (int64_t)k;
                if (k < rb) return total;
            }
        }
    }
    return total;
}

// pread exactly n bytes at off; returns bytes read
size_t pread_full(int fd, void *dst, size_t n, int64_t off)
{
    size_t got = 0;
    while (got < n) {
        const ssize_t k = pread(fd, static_cast<uint8_t *>(dst) + got, n - got, (off_t)(off + (int64_t)got));
        if (k <= 0) break;
        got += (size_t)k;
    }
    return got;
}

// Positional batch read: frames [r->frames, r->frames + n) by up to VCA_READ_THREADS (16) threads.  Returns VCA_OK
// or the error of the first failing frame (*first_bad = its batch index).
int read_positional(vca_reader *r, int n, void *const planes[3], const int64_t pitch[3], const int64_t fstride[3],
                    int *first_bad)
{
    const int fd = fileno(r->f);
    const vca_stream_info &in = r->info;
    // (frame index, status) of the first failing frame, packed into one word so that the
    // pair is updated atomically: index in the high 32 bits, status (as uint32) in the low 32;
    // an atomic min on the packed word keeps the lowest index together with its own status
    const uint64_t none = (uint64_t)(uint32_t)n << 32;
    std::atomic<uint64_t> first{none};
    auto fail = [&](int t, int rc) {
        const uint64_t mine = ((uint64_t)(uint32_t)t << 32) | (uint32_t)rc;
        uint64_t cur = first.load();
        while (mine < cur && !first.compare_exchange_weak(cur, mine)) {
        }
    };
    static const int kThreads = [] {
        const char *e = getenv("VCA_READ_THREADS");
        const int v = e ? atoi(e) : 16;
        return v < 1 ? 1 : (v > 64 ? 64 : v);
    }();
    const int T = std::max(1, std::min(n, kThreads));
    auto work = [&](int k) {
        for (int t = k; t < n; t += T) {
            int64_t off = r->data_off + (r->frames + t) * r->rec_bytes;
            if (r->y4m) {
                char m[6];
                const size_t km = pread_full(fd, m, 6, off);
                if (km < 6) {
                    fail(t, VCA_ERR_TRUNCATED_FRAME);
                    continue;
                }
                if (memcmp(m, "FRAME\n", 6) != 0) {
                    // "FRAME" + parameters: the records are not fixed-size after all
                    fail(t, memcmp(m, "FRAME", 5) == 0 && m[5] == ' ' ? VCA_IO_EOF : VCA_ERR_MALFORMED_FRAME_MARKER);
                    continue;
                }
                off += 6;
            }
            for (int p = 0; p < 3; ++p) {
                const int w = p ? in.chroma_width : in.width, h = p ? in.chroma_height : in.height;
                const size_t rb = (size_t)w * in.bytes_per_sample;
                uint8_t *base = static_cast<uint8_t *>(planes[p]) + (int64_t)t * fstride[p];
                bool ok = true;
                if ((size_t)pitch[p] == rb) {
                    ok = pread_full(fd, base, rb * h, off) == rb * h;
                } else {
                    for (int y = 0; y < h && ok; ++y)
                        ok = pread_full(fd, base + (int64_t)y * pitch[p], rb, off + (int64_t)y * rb) == rb;
                }
                if (!ok) {
                    fail(t, VCA_ERR_TRUNCATED_FRAME);
                    break;
                }
                off += (int64_t)rb * h;
            }
        }
    };
    std::thread pool[63];
    for (int k = 1; k < T; ++k) pool[k - 1] = std::thread(work, k);
    work(0);
    for (int k = 1; k < T; ++k) pool[k - 1].join();
    const uint64_t f = first.load();
    *first_bad = (int)(f >> 32);
    return f == none ? VCA_OK : (int)(uint32_t)(f & 0xFFFFFFFFu);
}

}  // namespace

extern "C" {

int vca_y4m_parse_header(const char *bytes, size_t len, vca_stream_info *info, size_t *header_len, int *warnings)
{
    if (!bytes || !info) return VCA_ERR_INVALID_ARG;
    static const char kMagic[] = "YUV4MPEG2";
    if (len < 9 || memcmp(bytes, kMagic, 9) != 0) return VCA_ERR_MALFORMED_MAGIC;
    const char *nl = (const char *)memchr(bytes, '\n', len);
    if (!nl) return VCA_ERR_MALFORMED_HEADER;
    if (nl > bytes + 9 && bytes[9] != ' ') return VCA_ERR_MALFORMED_MAGIC;  // "YUV4MPEG2X..."
    vca_stream_info in{};
    in.chroma_format = VCA_CHROMA_420;
    in.bit_depth = 8;
    in.frame_count = -1;
    bool haveW = false, haveH = false, haveF = false;
    int warn = 0;
    const char *p = bytes + 9;
    while (p < nl) {
        while (p < nl && *p == ' ') ++p;
        if (p >= nl) break;
        const char *e = p;
        while (e < nl && *e != ' ') ++e;
        const char tag = *p;
        const char *s = p + 1;
        long long a = 0, b = 0;
        switch (tag) {
        case 'W':
            if (!parse_int(s, e, &a)) return VCA_ERR_MALFORMED_HEADER;
            in.width = (int)a;
            haveW = true;
            break;
        case 'H':
            if (!parse_int(s, e, &a)) return VCA_ERR_MALFORMED_HEADER;
            in.height = (int)a;
            haveH = true;
            break;
        case 'F':
            if (!parse_ratio(s, e, &a, &b) || a <= 0 || b <= 0 || a > 0x7fffffff || b > 0x7fffffff)
                return VCA_ERR_MALFORMED_HEADER;
            in.fps_num = (int)a;
            in.fps_den = (int)b;
            haveF = true;
            break;
        case 'A':
            if (!parse_ratio(s, e, &a, &b)) return VCA_ERR_MALFORMED_HEADER;
            break;
        case 'I':
            if (e - s != 1) return VCA_ERR_MALFORMED_HEADER;
            if (*s != 'p') return VCA_ERR_INTERLACED;
            break;
        case 'C': {
            const std::string c(s, e);
            if (c == "420jpeg" || c == "420mpeg2" || c == "420paldv" || c == "420") {
                in.chroma_format = VCA_CHROMA_420;
                in.bit_depth = 8;
            } else if (c == "422") {
                in.chroma_format = VCA_CHROMA_422;
                in.bit_depth = 8;
            } else if (c == "444") {
                in.chroma_format = VCA_CHROMA_444;
                in.bit_depth = 8;
            } else if (c == "420p10" || c == "422p10" || c == "444p10") {
                in.chroma_format = c[1] == '2' && c[2] == '0' ? VCA_CHROMA_420
                                   : c[1] == '2'              ? VCA_CHROMA_422
                                                              : VCA_CHROMA_444;
                in.bit_depth = 10;
            } else if (c.size() > 4 && (c.compare(0, 4, "420p") == 0 || c.compare(0, 4, "422p") == 0 ||
                                        c.compare(0, 4, "444p") == 0)) {
                return VCA_ERR_UNSUPPORTED_BIT_DEPTH;  // p9, p12, p16, ...
            } else {
                return VCA_ERR_UNSUPPORTED_CHROMA;     // mono, 411, 444alpha, unknown
            }
            break;
        }
        case 'X':
            warn |= VCA_WARN_X_TOKENS;  // metadata: tolerated
            break;
        default:
            return VCA_ERR_MALFORMED_HEADER;
        }
        p = e;
    }
    if (!haveW || !haveH || !haveF) return VCA_ERR_MALFORMED_HEADER;
    int rc = finish_info(&in);
    if (rc) return rc;
    *info = in;
    if (header_len) *header_len = (size_t)(nl - bytes) + 1;
    if (warnings) *warnings = warn;
    return VCA_OK;
}

int vca_y4m_open(const char *path, vca_reader **out, vca_stream_info *info)
{
    if (!path || !out || !info) return VCA_ERR_INVALID_ARG;
    const bool is_stdin = strcmp(path, "-") == 0;
    FILE *f = is_stdin ? stdin : fopen(path, "rb");
    if (!f) return VCA_ERR_IO;
    char hdr[4096];
    size_t n = 0;
    int c;
    while (n < sizeof(hdr) && (c = fgetc(f)) != EOF) {  // header line only: never past its '\n'
        hdr[n++] = (char)c;
        if (c == '\n') break;
    }
    vca_stream_info in{};
    size_t hlen = 0;
    int warn = 0;
    int rc = vca_y4m_parse_header(hdr, n, &in, &hlen, &warn);
    if (rc) {
        if (!is_stdin) fclose(f);
        return rc;
    }
    if (!is_stdin) {
        const int64_t sz = file_size(f);
        const int64_t rec = 6 + in.frame_bytes;  // bare "FRAME\n" + payload
        if (sz >= (int64_t)hlen && (sz - (int64_t)hlen) % rec == 0) in.frame_count = (sz - (int64_t)hlen) / rec;
        setvbuf(f, nullptr, _IOFBF, 1 << 20);
    }
    vca_reader *r = new vca_reader;
    if (!is_stdin && in.frame_count >= 0) {  // bare "FRAME\n" markers (checked per frame on read)
        r->data_off = r->data_off_saved = (int64_t)hlen;
        r->rec_bytes = 6 + in.frame_bytes;
    }
    r->f = f;
    r->own = !is_stdin;
    r->y4m = true;
    r->info = in;
    r->warnings = warn;
    *info = in;
    *out = r;
    return VCA_OK;
}

int vca_raw_open(const char *path, int width, int height, int bit_depth, int chroma_format, vca_reader **out,
                 vca_stream_info *info)
{
    if (!path || !out || !info) return VCA_ERR_INVALID_ARG;
    vca_stream_info in{};
    in.width = width;
    in.height = height;
    in.bit_depth = bit_depth;
    in.chroma_format = chroma_format;
    in.frame_count = -1;
    int rc = finish_info(&in);
    if (rc) return rc;
    const bool is_stdin = strcmp(path, "-") == 0;
    FILE *f = is_stdin ? stdin : fopen(path, "rb");
    if (!f) return VCA_ERR_IO;
    vca_reader *r = new vca_reader;
    if (!is_stdin) {
        const int64_t sz = file_size(f);
        if (sz >= 0) {
            in.frame_count = sz / in.frame_bytes;
            if (sz % in.frame_bytes) r->warnings |= VCA_WARN_TRAILING_BYTES;  // discarded, reported
            r->data_off = 0;
            r->rec_bytes = in.frame_bytes;
        }
        setvbuf(f, nullptr, _IOFBF, 1 << 20);
    }
    r->f = f;
    r->own = !is_stdin;
    r->y4m = false;
    r->info = in;
    *info = in;
    *out = r;
    return VCA_OK;
}

int vca_reader_read(vca_reader *r, int max_frames, void *const planes[3], const int64_t pitch_bytes[3],
                    const int64_t frame_stride_bytes[3], int *n_read)
{
    if (!r || !planes || !pitch_bytes || !frame_stride_bytes || !n_read || max_frames < 0)
        return VCA_ERR_INVALID_ARG;
    *n_read = 0;
    for (int p = 0; p < 3; ++p) {
        const int w = p ? r->info.chroma_width : r->info.width;
        if (!planes[p] || pitch_bytes[p] < (int64_t)w * r->info.bytes_per_sample) return VCA_ERR_INVALID_ARG;
    }
    if (r->data_off >= 0 && r->info.frame_count >= 0) {  // regular file: parallel positional reads
        if (r->done) return VCA_IO_EOF;
        const int n = (int)std::min<int64_t>(max_frames, r->info.frame_count - r->frames);
        int first_bad = n;
        const int rc = n > 0 ? read_positional(r, n, planes, pitch_bytes, frame_stride_bytes, &first_bad) : VCA_OK;
        if (rc == VCA_IO_EOF) {
            // frame parameters after a bare-marker prefix: deliver the verified frames and
            // continue sequentially from the first parameterised record
            r->frames += first_bad;
            *n_read = first_bad;
            r->data_off = -1;
            r->info.frame_count = -1;
            if (fseeko(r->f, (off_t)(r->data_off_saved + r->frames * r->rec_bytes), SEEK_SET) != 0) return VCA_ERR_IO;
            return VCA_OK;
        }
        if (rc != VCA_OK) {  // the whole frames before the first bad one are delivered
            r->frames += first_bad;
            *n_read = first_bad;
            return rc;
        }
        r->frames += n;
        *n_read = n;
        if (n < max_frames) {
            r->done = true;
            return VCA_IO_EOF;
        }
        return VCA_OK;
    }
    for (int t = 0; t < max_frames; ++t) {
        if (r->done) return VCA_IO_EOF;
        if (!r->y4m && r->info.frame_count >= 0 && r->frames == r->info.frame_count) {
            r->done = true;  // a trailing partial frame (if any) is not read
            return VCA_IO_EOF;
        }
        if (r->y4m) {
            char m[6];
            const size_t k = read_full(r->f, m, 5);
            if (k == 0) {
                r->done = true;
                return VCA_IO_EOF;
            }
            if (k < 5 || memcmp(m, "FRAME", 5) != 0) return VCA_ERR_MALFORMED_FRAME_MARKER;
            int c;  // frame parameters (ignored) up to '\n'
            size_t guard = 0;
            while ((c = fgetc(r->f)) != EOF && c != '\n') {
                if (++guard > 4096) return VCA_ERR_MALFORMED_FRAME_MARKER;
            }
            if (c == EOF) return VCA_ERR_TRUNCATED_FRAME;
        }
        const int64_t got = read_payload(r, planes, pitch_bytes, frame_stride_bytes, t);
        if (got < r->info.frame_bytes) {
            if (!r->y4m) {  // raw stream without a known size: trailing partial frame
                r->done = true;
                if (got > 0) r->warnings |= VCA_WARN_TRAILING_BYTES;
                return VCA_IO_EOF;
            }
            return VCA_ERR_TRUNCATED_FRAME;
        }
        ++r->frames;
        ++*n_read;
    }
    return VCA_OK;
}

int64_t vca_reader_frames(const vca_reader *r) { return r ? r->frames : -1; }
int vca_reader_warnings(const vca_reader *r) { return r ? r->warnings : 0; }

void vca_reader_close(vca_reader *r)
{
    if (!r) return;
    if (r->own && r->f) fclose(r->f);
    delete r;
}

// ---------------------------------------------------------------- streaming driver
int vca_analyze_stream(vca_ctx *ctx, vca_reader *r, int batch_frames, vca_features *out_host, int64_t capacity,
                       int64_t *n_out, double *seconds)
{
    if (!ctx || !r || !out_host || !n_out || capacity < 1) return VCA_ERR_INVALID_ARG;
    *n_out = 0;
    if (seconds) *seconds = 0.0;
    vca_info ci;
    int rc = vca_get_info(ctx, &ci);
    if (rc) return rc;
    const vca_stream_info &in = r->info;
    if (in.chroma_format != VCA_CHROMA_420 || in.width != ci.width || in.height != ci.height ||
        in.bit_depth != ci.bit_depth)
        return VCA_ERR_GEOMETRY;
    if (batch_frames <= 0) batch_frames = 32;
    if (batch_frames > capacity) batch_frames = (int)capacity;

    // pinned batches, rows padded to 16 bytes (vca_analyze_host's alignment rule)
    int64_t pitch[3], fstride[3], off[3];
    int64_t fbytes = 0;
    for (int p = 0; p < 3; ++p) {
        const int w = p ? in.chroma_width : in.width, h = p ? in.chroma_height : in.height;
        pitch[p] = ((int64_t)w * in.bytes_per_sample + 15) & ~(int64_t)15;
        fstride[p] = pitch[p] * h;
        off[p] = fbytes * batch_frames;
        fbytes += fstride[p];
    }
    uint8_t *buf[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b) {
        if (cudaHostAlloc(reinterpret_cast<void **>(&buf[b]), (size_t)fbytes * batch_frames, cudaHostAllocDefault) !=
            cudaSuccess) {
            cudaGetLastError();
            if (buf[0]) cudaFreeHost(buf[0]);
            return VCA_ERR_OOM;
        }
    }
    // two-slot hand-off between the reader thread and the analysing (calling) thread
    std::mutex mu;
    std::condition_variable cv;
    int filled_n[2] = {0, 0}, filled_rc[2] = {0, 0};
    bool full[2] = {false, false};
    bool stop = false;
    const auto t0 = std::chrono::steady_clock::now();
    std::thread reader([&] {
        int64_t requested = 0;
        for (int k = 0;; ++k) {
            const int b = k & 1;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return !full[b] || stop; });
                if (stop) return;
            }
            const int want = (int)((capacity - requested) < batch_frames ? (capacity - requested) : batch_frames);
            void *pl[3] = {buf[b] + off[0], buf[b] + off[1], buf[b] + off[2]};
            int n = 0;
            int rrc = want > 0 ? vca_reader_read(r, want, pl, pitch, fstride, &n) : VCA_OK;
            requested += n;
            {
                std::lock_guard<std::mutex> lk(mu);
                filled_n[b] = n;
                filled_rc[b] = rrc;
                full[b] = true;
            }
            cv.notify_all();
            if (rrc != VCA_OK || requested >= capacity) return;
        }
    });
    int result = VCA_OK;
    for (int k = 0;; ++k) {
        const int b = k & 1;
        int n, rrc;
        {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return full[b]; });
            n = filled_n[b];
            rrc = filled_rc[b];
        }
        if (n > 0) {
            const void *pl[3] = {buf[b] + off[0], buf[b] + off[1], buf[b] + off[2]};
            int arc = vca_analyze_host(ctx, pl, pitch, fstride, n, 0, 8, out_host + *n_out, nullptr);
            if (arc) {
                result = arc;
                break;
            }
            *n_out += n;
        }
        {
            std::lock_guard<std::mutex> lk(mu);
            full[b] = false;
        }
        cv.notify_all();
        if (rrc != VCA_OK) {
            result = rrc;
            break;
        }
        if (*n_out >= capacity) break;
    }
    {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
    }
    cv.notify_all();
    reader.join();
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    cudaFreeHost(buf[0]);
    cudaFreeHost(buf[1]);
    return result;
}

// ---------------------------------------------------------------- CSV / summary
int64_t vca_write_csv(const char *path, const vca_features *rec, int64_t n)
{
    if (!path || n < 0 || (n > 0 && !rec)) return VCA_ERR_INVALID_ARG;
    const bool to_stdout = strcmp(path, "-") == 0;
    FILE *f = to_stdout ? stdout : fopen(path, "wb");
    if (!f) return VCA_ERR_IO;
    // '.' decimal separator whatever the process locale
    locale_t cl = newlocale(LC_NUMERIC_MASK, "C", (locale_t)0);
    locale_t old = cl ? uselocale(cl) : (locale_t)0;
    int64_t bytes = 0;
    bool ok = true;
    int k = fprintf(f, "POC,E_Y,h,L_Y,E_U,L_U,E_V,L_V\n");
    if (k < 0) ok = false;
    bytes += k;
    for (int64_t i = 0; ok && i < n; ++i) {
        const vca_features &r = rec[i];
        k = fprintf(f, "%lld,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f,%.6f\n", (long long)r.poc, r.E_Y, r.h, r.L_Y, r.E_U, r.L_U,
                    r.E_V, r.L_V);
        if (k < 0) ok = false;
        bytes += k;
    }
    if (cl) {
        uselocale(old);
        freelocale(cl);
    }
    if (to_stdout) {
        if (fflush(f) != 0) ok = false;
    } else if (fclose(f) != 0) {
        ok = false;
    }
    return ok ? bytes : VCA_ERR_IO;
}

int vca_summarize(const vca_features *rec, int64_t n, double mean[7], double max[7])
{
    if (!rec || n < 1 || !mean || !max) return VCA_ERR_INVALID_ARG;
    double s[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < 7; ++j) max[j] = -1.0 / 0.0;
    for (int64_t i = 0; i < n; ++i) {  // POC order
        const double v[7] = {rec[i].E_Y, rec[i].h, rec[i].L_Y, rec[i].E_U, rec[i].L_U, rec[i].E_V, rec[i].L_V};
        for (int j = 0; j < 7; ++j) {
            s[j] += v[j];
            if (v[j] > max[j]) max[j] = v[j];
        }
    }
    for (int j = 0; j < 7; ++j) mean[j] = s[j] / (double)n;
    return VCA_OK;
}

}  // extern "C"
