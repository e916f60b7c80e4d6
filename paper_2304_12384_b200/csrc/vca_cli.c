/*
 * vca_cli.c -- a native command-line client of the C ABI (include/vca.h, include/vca_io.h):
 * no Python, no PyTorch.  Streams a Y4M file (or '-') or a raw YUV file through libvca and
 * writes the per-frame features CSV (S:456 format) -- the same operation as
 * `python -m paper_2304_12384_b200.cli analyze`, showing the boundary is usable from plain C.
 *
 *   vca_cli INPUT.y4m [-o OUT.csv] [--block N] [--low-pass] [--batch N]
 *   vca_cli INPUT.yuv --width W --height H [--bit-depth 8|10] [-o OUT.csv] ...
 *
 * Exit codes: 0 success, 1 usage error, 2 input / runtime error.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/vca.h"
#include "../../include/vca_io.h"

static int usage(const char *msg)
{
    fprintf(stderr, "usage error: %s\n"
                    "usage: vca_cli INPUT [-o OUT.csv] [--width W --height H --bit-depth B] [--block N]"
                    " [--low-pass] [--batch N]\n",
            msg);
    return 1;
}

static int fail(const char *what, int rc)
{
    fprintf(stderr, "input error: %s: %s (%d)\n", what, vca_status_string(rc), rc);
    return 2;
}

int main(int argc, char **argv)
{
    const char *in = NULL, *out = "-";
    int width = 0, height = 0, bd = 8, block = 0, lowpass = 0, batch = 32;
    for (int i = 1; i < argc; ++i) {
        const char *a = argv[i];
        if (!strcmp(a, "-o") && i + 1 < argc) out = argv[++i];
        else if (!strcmp(a, "--width") && i + 1 < argc) width = atoi(argv[++i]);
        else if (!strcmp(a, "--height") && i + 1 < argc) height = atoi(argv[++i]);
        else if (!strcmp(a, "--bit-depth") && i + 1 < argc) bd = atoi(argv[++i]);
        else if (!strcmp(a, "--block") && i + 1 < argc) block = atoi(argv[++i]);
        else if (!strcmp(a, "--batch") && i + 1 < argc) batch = atoi(argv[++i]);
        else if (!strcmp(a, "--low-pass")) lowpass = 1;
        else if (a[0] == '-' && a[1] != '\0') return usage("unknown flag");
        else if (!in) in = a;
        else return usage("more than one input");
    }
    if (!in) return usage("missing input");
    const char *dot = strrchr(in, '.');
    const int y4m = !strcmp(in, "-") || (dot && !strcmp(dot, ".y4m"));
    if (!y4m && (width <= 0 || height <= 0)) return usage("raw input needs --width and --height");

    vca_reader *r = NULL;
    vca_stream_info info;
    int rc = y4m ? vca_y4m_open(in, &r, &info) : vca_raw_open(in, width, height, bd, VCA_CHROMA_420, &r, &info);
    if (rc) return fail("open", rc);
    vca_ctx *ctx = NULL;
    rc = vca_create(info.width, info.height, info.bit_depth, info.chroma_format, block, lowpass, &ctx);
    if (rc) {
        vca_reader_close(r);
        return fail("vca_create", rc);
    }
    int64_t cap = info.frame_count > 0 ? info.frame_count : 1024, n = 0;
    vca_features *rec = (vca_features *)malloc(sizeof(vca_features) * (size_t)cap);
    double secs = 0.0;
    for (;;) {
        int64_t got = 0;
        double s = 0.0;
        if (n == cap) {
            cap *= 2;
            vca_features *grown = (vca_features *)realloc(rec, sizeof(vca_features) * (size_t)cap);
            if (!grown) {
                rc = VCA_ERR_OOM;
                break;
            }
            rec = grown;
        }
        rc = vca_analyze_stream(ctx, r, batch, rec + n, cap - n, &got, &s);
        n += got;
        secs += s;
        if (rc != VCA_OK) break;
    }
    if (rc == VCA_IO_EOF) rc = VCA_OK;
    if (rc == VCA_OK && n == 0) rc = VCA_ERR_INVALID_ARG; /* EmptyStream */
    if (rc == VCA_OK && vca_write_csv(out, rec, n) < 0) rc = VCA_ERR_IO;
    if (rc == VCA_OK) fprintf(stderr, "# frames=%lld seconds=%.6f fps=%.2f\n", (long long)n, secs, secs > 0 ? n / secs : 0.0);
    free(rec);
    vca_destroy(ctx);
    vca_reader_close(r);
    return rc == VCA_OK ? 0 : fail("analysis", rc);
}
