/*
 * ORACLE (test infrastructure only — never linked into the product).
 *
 * Plain-C restatement of the reference CPU engine for the five BASELINE
 * configurations, one straight loop nest per abstraction node, materialising
 * every intermediate exactly like run_naive does.  Used by tests/ as the
 * parity checker and by bench.py as the portable CPU baseline ("kind":
 * "port").  Pinned against the reference itself (oracle/_ref, built from
 * /root/reference by oracle/Makefile) and the golden fixtures in
 * tests/golden/ (tests/test_oracle.py).
 *
 * Reference semantics followed (ref = /root/reference/proj):
 *   Clamp window reads               src/execute.cpp:233-245
 *   Sum combine, row-major, int64    src/execute.cpp:560-599
 *   cast_value Saturate (llround)    src/expr.cpp:8-43
 *   Gaussian3x3 mask / post          src/registry.cpp:722-746 (1/16 double)
 *   Sobel3x3 masks, sat S16          src/registry.cpp:748-784
 *   Magnitude sqrt(double)           src/registry.cpp:555-575
 *   Multiply -> S32                  src/registry.cpp:456-487
 *   Box3x3 (1/9 double)              src/registry.cpp:703-720
 *   Subtract / Add -> S16            src/registry.cpp:119-129, 456-487
 *   ConvertDepth (saturate)          src/registry.cpp:642-670
 *   Convolve (scale -> 1/scale)      src/registry.cpp:837-878
 *   Histogram bin formula            src/registry.cpp:882-913
 *   MeanStdDev finalize              src/registry.cpp:957-1010
 * Compiled with -ffp-contract=off so double expressions are not fused.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int64_t clampi64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* cast_value(T, Saturate, real r) for integer T (src/expr.cpp:15-24, 34). */
static int64_t sat_real(double r, int64_t lo, int64_t hi) {
    if (isnan(r)) return 0;
    if (r >= (double)hi) return hi;
    if (r <= (double)lo) return lo;
    return clampi64(llround(r), lo, hi);
}

/* 3x3 Sum window of mask * in over an int32 plane with Clamp borders. */
static int64_t win3(const int32_t* src, int w, int h, int x, int y, const int m[9]) {
    int64_t s = 0;
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            int xx = clampi(x + dx, 0, w - 1), yy = clampi(y + dy, 0, h - 1);
            s += (int64_t)m[(dy + 1) * 3 + dx + 1] * src[(size_t)yy * w + xx];
        }
    return s;
}

static int32_t* widen_u8(const uint8_t* in, int w, int h) {
    int32_t* p = (int32_t*)malloc(sizeof(int32_t) * (size_t)w * h);
    for (size_t i = 0; i < (size_t)w * h; ++i) p[i] = in[i];
    return p;
}

static const int kGauss[9] = {1, 2, 1, 2, 4, 2, 1, 2, 1};
static const int kSobelX[9] = {-1, 0, 1, -2, 0, 2, -1, 0, 1};
static const int kSobelY[9] = {-1, -2, -1, 0, 0, 0, 1, 2, 1};
static const int kBox[9] = {1, 1, 1, 1, 1, 1, 1, 1, 1};

/* Gaussian3x3 on U8 -> U8 (int32 plane). */
void gvxo_gaussian3x3(const int32_t* in, int w, int h, int32_t* out) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            out[(size_t)y * w + x] = (int32_t)sat_real((double)win3(in, w, h, x, y, kGauss) * (1.0 / 16.0), 0, 255);
}

/* Sobel3x3 -> S16 gx, gy (sat_S16 of the integer sum). */
void gvxo_sobel3x3(const int32_t* in, int w, int h, int32_t* gx, int32_t* gy) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            size_t i = (size_t)y * w + x;
            if (gx) gx[i] = (int32_t)clampi64(win3(in, w, h, x, y, kSobelX), -32768, 32767);
            if (gy) gy[i] = (int32_t)clampi64(win3(in, w, h, x, y, kSobelY), -32768, 32767);
        }
}

/* Magnitude: sat_S16(llround(sqrt(double(gx*gx + gy*gy)))). */
void gvxo_magnitude(const int32_t* gx, const int32_t* gy, size_t n, int32_t* out) {
    for (size_t i = 0; i < n; ++i) {
        int64_t s = (int64_t)gx[i] * gx[i] + (int64_t)gy[i] * gy[i];
        out[i] = (int32_t)sat_real(sqrt((double)s), -32768, 32767);
    }
}

/* cfg1 / cfg5: U8 -> S16 magnitude. */
void gvxo_edge(const uint8_t* in, int w, int h, int16_t* mag) {
    size_t n = (size_t)w * h;
    int32_t* src = widen_u8(in, w, h);
    int32_t* g = (int32_t*)malloc(sizeof(int32_t) * n);
    int32_t* gx = (int32_t*)malloc(sizeof(int32_t) * n);
    int32_t* gy = (int32_t*)malloc(sizeof(int32_t) * n);
    int32_t* m = (int32_t*)malloc(sizeof(int32_t) * n);
    gvxo_gaussian3x3(src, w, h, g);
    gvxo_sobel3x3(g, w, h, gx, gy);
    gvxo_magnitude(gx, gy, n, m);
    for (size_t i = 0; i < n; ++i) mag[i] = (int16_t)m[i];
    free(src), free(g), free(gx), free(gy), free(m);
}

/* cfg2: Harris mask (and optionally the F32 response). */
void gvxo_harris(const uint8_t* in, int w, int h, double k, double threshold, uint8_t* mask, float* resp_out) {
    size_t n = (size_t)w * h;
    int32_t* src = widen_u8(in, w, h);
    int32_t *gx = malloc(4 * n), *gy = malloc(4 * n);
    int32_t *pxx = malloc(4 * n), *pyy = malloc(4 * n), *pxy = malloc(4 * n);
    int32_t *sxx = malloc(4 * n), *syy = malloc(4 * n), *sxy = malloc(4 * n);
    gvxo_sobel3x3(src, w, h, gx, gy);
    for (size_t i = 0; i < n; ++i) { /* Multiply: sat_S32(a * b) */
        pxx[i] = (int32_t)clampi64((int64_t)gx[i] * gx[i], INT32_MIN, INT32_MAX);
        pyy[i] = (int32_t)clampi64((int64_t)gy[i] * gy[i], INT32_MIN, INT32_MAX);
        pxy[i] = (int32_t)clampi64((int64_t)gx[i] * gy[i], INT32_MIN, INT32_MAX);
    }
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) { /* Box3x3 on S32: sat_S32(llround(s * (1/9))) */
            size_t i = (size_t)y * w + x;
            sxx[i] = (int32_t)sat_real((double)win3(pxx, w, h, x, y, kBox) * (1.0 / 9.0), INT32_MIN, INT32_MAX);
            syy[i] = (int32_t)sat_real((double)win3(pyy, w, h, x, y, kBox) * (1.0 / 9.0), INT32_MIN, INT32_MAX);
            sxy[i] = (int32_t)sat_real((double)win3(pxy, w, h, x, y, kBox) * (1.0 / 9.0), INT32_MIN, INT32_MAX);
        }
    for (size_t i = 0; i < n; ++i) {
        /* HarrisResponse: F32((a*b - c*c) - k*((a+b)*(a+b))), int64 then double */
        int64_t det = (int64_t)sxx[i] * syy[i] - (int64_t)sxy[i] * sxy[i];
        int64_t tr = (int64_t)sxx[i] + syy[i];
        double r = (double)det - k * (double)(tr * tr);
        float rf = (float)r;
        if (resp_out) resp_out[i] = rf;
        /* ThresholdF32: sat_U8(resp > T ? 255 : 0) */
        mask[i] = ((double)rf > threshold) ? 255 : 0;
    }
    free(src), free(gx), free(gy), free(pxx), free(pyy), free(pxy), free(sxx), free(syy), free(sxy);
}

/* Linear KxK Sum window with Clamp over an int32 plane. */
static int64_t wink(const int32_t* src, int w, int h, int x, int y, const int* m, int ks) {
    int r = ks / 2;
    int64_t s = 0;
    for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx) {
            int xx = clampi(x + dx, 0, w - 1), yy = clampi(y + dy, 0, h - 1);
            s += (int64_t)m[(dy + r) * ks + dx + r] * src[(size_t)yy * w + xx];
        }
    return s;
}

static const int kBinomial5[25] = {1, 4, 6, 4, 1, 4, 16, 24, 16, 4, 6, 24, 36, 24, 6, 4, 16, 24, 16, 4, 1, 4, 6, 4, 1};

/* cfg3: Blur5x5 (user local, sat_U8(s * (1/256))) -> Subtract -> Add -> ConvertDepth. */
void gvxo_unsharp(const uint8_t* in, int w, int h, uint8_t* out) {
    size_t n = (size_t)w * h;
    int32_t* src = widen_u8(in, w, h);
    int32_t* blur = malloc(4 * n);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            blur[(size_t)y * w + x] =
                (int32_t)sat_real((double)wink(src, w, h, x, y, kBinomial5, 5) * (1.0 / 256.0), 0, 255);
    for (size_t i = 0; i < n; ++i) {
        int64_t diff = clampi64((int64_t)src[i] - blur[i], -32768, 32767); /* Subtract -> S16 */
        int64_t sum = clampi64((int64_t)src[i] + diff, -32768, 32767);     /* Add -> S16 */
        out[i] = (uint8_t)clampi64(sum, 0, 255);                            /* ConvertDepth -> U8 */
    }
    free(src), free(blur);
}

/* cfg4 (one frame): Convolve(binomial5, scale 256) -> S16 -> ConvertDepth -> U8
 * -> Histogram(256, 0, 256) + MeanStdDev. */
void gvxo_conv_stats(const uint8_t* in, int w, int h, long long* hist, double* mean, double* stddev) {
    size_t n = (size_t)w * h;
    int32_t* src = widen_u8(in, w, h);
    int64_t sum = 0, sumsq = 0;
    for (int b = 0; b < 256; ++b) hist[b] = 0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int64_t c = sat_real((double)wink(src, w, h, x, y, kBinomial5, 5) * (1.0 / 256.0), -32768, 32767);
            int64_t u = clampi64(c, 0, 255);
            int64_t bin = ((u - 0) * 256) / 256;
            if (bin >= 0 && bin < 256) hist[bin] += 1;
            sum += u;
            sumsq += u * u;
        }
    /* reduce_mean finalize: F32((sum * 1.0) / n) */
    double m = (double)(float)(((double)sum * 1.0) / (double)(int64_t)n);
    /* reduce_stddev finalize: F32(sqrt(max((sumsq * 1.0) / n - m*m, 0))) with m the F32 mean */
    double var = ((double)sumsq * 1.0) / (double)(int64_t)n - m * m;
    if (var < 0.0) var = 0.0;
    *mean = m;
    *stddev = (double)(float)sqrt(var);
    free(src);
}

/* Generalised forms of the cfg3 / cfg4 chains for the C-ABI kernels
 * (gvxb_stencil_point / gvxb_conv_stats) over any KxK integer mask and
 * divisor d: the local node post body sat_T(s * (1.0 / d)) (a user local
 * node, or Convolve with scale d, src/registry.cpp:837-878), then
 *   mode 0: the U8 result;  mode 1: Subtract -> Add -> ConvertDepth.
 */
void gvxo_stencil_u8(const uint8_t* in, int w, int h, int k, const int* mask, long long d, int mode,
                     uint8_t* out) {
    size_t n = (size_t)w * h;
    int32_t* src = widen_u8(in, w, h);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            size_t i = (size_t)y * w + x;
            int64_t b = sat_real((double)wink(src, w, h, x, y, mask, k) * (1.0 / (double)d), 0, 255);
            if (mode == 0) {
                out[i] = (uint8_t)b;
            } else {
                int64_t diff = clampi64((int64_t)src[i] - b, -32768, 32767);
                int64_t sum = clampi64((int64_t)src[i] + diff, -32768, 32767);
                out[i] = (uint8_t)clampi64(sum, 0, 255);
            }
        }
    (void)n;
    free(src);
}

/* Convolve(mask, scale) -> conv format [lo, hi] -> ConvertDepth(U8, shift,
 * policy: Shr then Saturate / Wrap, src/registry.cpp:642-670) -> Histogram
 * (bins, offset, range; bin = ((v - offset) * bins) / range truncating,
 * out-of-range skipped, src/execute.cpp:698-727) + MeanStdDev.  `conv`
 * (optional) receives the U8 image. */
void gvxo_conv_stats_ex(const uint8_t* in, int w, int h, int k, const int* mask, long long scale, int conv_lo,
                        int conv_hi, int shift, int wrap, int bins, long long offset, long long range,
                        long long* hist, double* mean, double* stddev, uint8_t* conv) {
    size_t n = (size_t)w * h;
    int32_t* src = widen_u8(in, w, h);
    int64_t sum = 0, sumsq = 0;
    for (int b = 0; b < bins; ++b) hist[b] = 0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int64_t c = sat_real((double)wink(src, w, h, x, y, mask, k) * (1.0 / (double)scale), conv_lo, conv_hi);
            if (shift > 0) c >>= shift;
            int64_t u = wrap ? (c & 0xFF) : clampi64(c, 0, 255);
            if (conv) conv[(size_t)y * w + x] = (uint8_t)u;
            int64_t t = (u - offset) * bins;
            int64_t bin = t / range;
            if (bin >= 0 && bin < bins) hist[bin] += 1;
            sum += u;
            sumsq += u * u;
        }
    double m = (double)(float)(((double)sum * 1.0) / (double)(int64_t)n);
    double var = ((double)sumsq * 1.0) / (double)(int64_t)n - m * m;
    if (var < 0.0) var = 0.0;
    *mean = m;
    *stddev = (double)(float)sqrt(var);
    free(src);
}
