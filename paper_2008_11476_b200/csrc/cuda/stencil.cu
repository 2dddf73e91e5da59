// K3 — linear KxK integer stencil over U8 fused with its point consumers
// (cfg3: user-defined 5x5 blur -> Subtract -> Add -> ConvertDepth), and
// K4 — KxK convolution -> ConvertDepth -> {Histogram, sum, sum of squares}
// with the MeanStdDev finalize (cfg4).
//
// Exactness contract:
//   local post body sat_T(llround(s * (1/d))) == sat_T(round_half_away(s/d))
//   when d is a power of two (exact product) or d is odd with |s| < 2^50
//   (the host lowering only selects these kernels under those proofs);
//   point chains use the reference's per-node saturation at every boundary;
//   histogram bin ((v - offset) * bins) / range truncates toward zero and
//   skips out-of-range bins (ref:src/registry.cpp:882-913,
//   ref:src/execute.cpp:698-727); sums are exact int64;
//   MeanStdDev finalize in IEEE double without contraction, in the
//   reference's operation order (ref:src/registry.cpp:957-1010).
#include "packed.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace gvxd {

constexpr int kStThreads = 128;
constexpr int kStTW = 4 * kStThreads;
constexpr int kStTH = 32;
constexpr int kStSW = kStTW + 64;
constexpr int kStBox = 192;

struct StencilParams {
    int width;
    Band band;
    int mask[49];
    int div;       // round-half-away divisor (1 = none)
    int out_lo, out_hi; // saturation range of the stencil node's output type
    int mode;
    uint8_t* dst;
    int64_t dst_pitch, dst_fstride;
};

/// 4 + 2R source bytes starting at column c - R (R <= 3) from aligned words.
template <int R>
__device__ __forceinline__ void fetch_span(const uint8_t* row, int off, int (&a)[4 + 2 * R]) {
    const uint32_t wl = lds32(row, off - 4), wc = lds32(row, off), wr = lds32(row, off + 4);
#pragma unroll
    for (int k = 0; k < R; ++k) a[k] = byte_of(wl, 4 - R + k);
#pragma unroll
    for (int k = 0; k < 4; ++k) a[R + k] = byte_of(wc, k);
#pragma unroll
    for (int k = 0; k < R; ++k) a[R + 4 + k] = byte_of(wr, k);
}

template <int K>
__device__ __forceinline__ void stencil_sums(const uint8_t* tile, int row_j, int off, const int* mask,
                                             int (&acc)[4]) {
    constexpr int R = K / 2;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = 0;
#pragma unroll
    for (int dy = 0; dy < K; ++dy) {
        int a[4 + 2 * R];
        fetch_span<R>(tile + (row_j + dy) * kStSW, off, a);
#pragma unroll
        for (int dx = 0; dx < K; ++dx) {
            const int m = mask[dy * K + dx];
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] += m * a[i + dx];
        }
    }
}

__device__ __forceinline__ int apply_div(int s, int d) { return d == 1 ? s : round_div_away(s, d); }

template <int K, int kMode>
__global__ void __launch_bounds__(kStThreads) stencil_point_kernel(const __grid_constant__ CUtensorMap map,
                                                                   StencilParams p) {
    constexpr int R = K / 2;
    constexpr int SH = kStTH + 2 * R;
    __shared__ alignas(128) uint8_t tile[SH * kStSW];
    __shared__ uint64_t bar;

    const int x0 = blockIdx.x * kStTW;
    const int y0 = p.band.row0 + blockIdx.y * kStTH;
    const int y1 = min(y0 + kStTH, p.band.row1);
    const int frame = blockIdx.z;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    stage_tile_u8<kStSW, SH>(tile, &map, &bar, x0 - 32, y0 - R, frame, p.width, p.band);

    const int c = x0 + 4 * static_cast<int>(threadIdx.x);
    if (c >= p.width) return;
    const int off = 4 * static_cast<int>(threadIdx.x) + 32;
    uint8_t* base = p.dst + frame * p.dst_fstride;

    for (int y = y0; y < y1; ++y) {
        const int j = y - y0; // smem row of the window top
        int acc[4];
        stencil_sums<K>(tile, j, off, p.mask, acc);
        const uint32_t centre = lds32(tile + (j + R) * kStSW, off);
        uint32_t packed = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int b = clampi(apply_div(acc[i], p.div), p.out_lo, p.out_hi);
            int v;
            if (kMode == 0) {
                v = b;
            } else {
                const int x = byte_of(centre, i);
                const int diff = sat_s16(x - b); // Subtract(in, blur) -> S16
                const int sum = sat_s16(x + diff); // Add(in, diff) -> S16
                v = sat_u8(sum);                   // ConvertDepth(S16 -> U8)
            }
            packed |= static_cast<uint32_t>(v & 0xFF) << (8 * i);
        }
        uint8_t* dp = base + static_cast<int64_t>(y - p.band.dst_row0) * p.dst_pitch + c;
        if (c + 3 < p.width) {
            *reinterpret_cast<uint32_t*>(dp) = packed;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (c + i < p.width) dp[i] = static_cast<uint8_t>(packed >> (8 * i));
        }
    }
}

// ---------------------------------------------------------------- K4

struct ConvStatsParams {
    int width, height;
    Band band;
    int mask[49];
    int div;
    int conv_lo, conv_hi; // saturation range of the convolve output format
    int shift;            // ConvertDepth right shift (0 = none)
    int wrap;             // ConvertDepth policy: 0 saturate, 1 wrap (to U8)
    int bins;
    long long offset, range;
    int identity_bins;    // offset == 0 && bins == range
    uint8_t* conv_out;
    int64_t conv_pitch, conv_fstride;
    gvxb_value* hist; // frames x bins (integer Value slots)
    unsigned long long* sum;
    unsigned long long* sumsq;
    // one-launch form: as SepParams::acc (publish_if_last)
    unsigned long long* acc;
    int ctas_per_frame;
    long long npx;
    gvxb_value* mean;
    gvxb_value* stddev;
};

__device__ __forceinline__ void meanstd_of(unsigned long long s1, unsigned long long s2, long long n, gvxb_value* mean,
                                           gvxb_value* sd);

/// One-launch conv+stats epilogue, called by every thread of a CTA after its
/// histogram / sum atomics: the frame's last CTA to finish (every CTA fences
/// its atomics before counting itself done) moves the accumulated histogram
/// into the output slots, derives MeanStdDev, and leaves the accumulators,
/// sums and counter zero for the next execution.
__device__ __forceinline__ void publish_if_last(int frame, int tid, int nt, int bins, unsigned long long* acc_all,
                                                gvxb_value* hist, unsigned long long* sum, unsigned long long* sumsq,
                                                int ctas_per_frame, long long npx, gvxb_value* mean, gvxb_value* sd) {
    __shared__ int last;
    __threadfence();
    __syncthreads();
    unsigned long long* acc = acc_all + static_cast<int64_t>(frame) * (bins + 1);
    if (tid == 0) last = atomicAdd(acc + bins, 1ull) == static_cast<unsigned long long>(ctas_per_frame - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (hist) {
        for (int b = tid; b < bins; b += nt) {
            gvxb_value& h = hist[static_cast<int64_t>(frame) * bins + b];
            h.real = 0;
            h.bits = static_cast<long long>(atomicExch(acc + b, 0ull));
        }
    }
    if (tid == 0) {
        const unsigned long long t1 = atomicExch(&sum[frame], 0ull), t2 = atomicExch(&sumsq[frame], 0ull);
        meanstd_of(t1, t2, npx, mean ? mean + frame : nullptr, sd ? sd + frame : nullptr);
        atomicExch(acc + bins, 0ull);
    }
}

template <int K>
__global__ void __launch_bounds__(kStThreads) conv_stats_kernel(const __grid_constant__ CUtensorMap map,
                                                                ConvStatsParams p) {
    constexpr int R = K / 2;
    constexpr int SH = kStTH + 2 * R;
    constexpr int kWarps = kStThreads / 32;
    __shared__ alignas(128) uint8_t tile[SH * kStSW];
    __shared__ uint64_t bar;
    extern __shared__ unsigned hist_smem[]; // kWarps x bins

    const int x0 = blockIdx.x * kStTW;
    const int y0 = p.band.row0 + blockIdx.y * kStTH;
    const int y1 = min(y0 + kStTH, p.band.row1);
    const int frame = blockIdx.z;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < kWarps * p.bins; i += blockDim.x) hist_smem[i] = 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    stage_tile_u8<kStSW, SH>(tile, &map, &bar, x0 - 32, y0 - R, frame, p.width, p.band);

    const int c = x0 + 4 * static_cast<int>(threadIdx.x);
    const int off = 4 * static_cast<int>(threadIdx.x) + 32;
    unsigned* my_hist = hist_smem + warp * p.bins;
    unsigned lsum = 0, lsq = 0;
    if (c < p.width) {
        uint8_t* base = p.conv_out ? p.conv_out + frame * p.conv_fstride : nullptr;
        for (int y = y0; y < y1; ++y) {
            int acc[4];
            stencil_sums<K>(tile, y - y0, off, p.mask, acc);
            uint32_t packed = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (c + i >= p.width) continue;
                int v = clampi(apply_div(acc[i], p.div), p.conv_lo, p.conv_hi); // Convolve -> S16
                if (p.shift > 0) v >>= p.shift;                                 // ConvertDepth shift
                v = p.wrap ? (v & 0xFF) : sat_u8(v);                             // -> U8
                packed |= static_cast<uint32_t>(v) << (8 * i);
                lsum += static_cast<unsigned>(v);
                lsq += static_cast<unsigned>(v * v);
                int bin;
                if (p.identity_bins) {
                    bin = v;
                } else {
                    const long long t = (static_cast<long long>(v) - p.offset) * p.bins;
                    bin = static_cast<int>(t / p.range);
                    if (t / p.range < 0 || t / p.range >= p.bins) bin = -1;
                }
                if (bin >= 0 && bin < p.bins) atomicAdd(&my_hist[bin], 1u);
            }
            if (base) {
                uint8_t* dp = base + static_cast<int64_t>(y - p.band.dst_row0) * p.conv_pitch + c;
                if (c + 3 < p.width) {
                    *reinterpret_cast<uint32_t*>(dp) = packed;
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (c + i < p.width) dp[i] = static_cast<uint8_t>(packed >> (8 * i));
                }
            }
        }
    }
    // block reduction of the sums (per-thread values fit in 32 bits)
    unsigned long long s = lsum, q = lsq;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    __shared__ unsigned long long red[2][kWarps];
    if ((threadIdx.x & 31) == 0) {
        red[0][warp] = s;
        red[1][warp] = q;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long ts = 0, tq = 0;
        for (int w = 0; w < kWarps; ++w) {
            ts += red[0][w];
            tq += red[1][w];
        }
        atomicAdd(&p.sum[frame], ts);
        atomicAdd(&p.sumsq[frame], tq);
    }
    if (p.hist) {
        for (int b = threadIdx.x; b < p.bins; b += blockDim.x) {
            unsigned t = 0;
            for (int w = 0; w < kWarps; ++w) t += hist_smem[w * p.bins + b];
            unsigned long long* slot =
                p.acc ? p.acc + static_cast<int64_t>(frame) * (p.bins + 1) + b
                      : reinterpret_cast<unsigned long long*>(&p.hist[static_cast<int64_t>(frame) * p.bins + b].bits);
            if (t) atomicAdd(slot, static_cast<unsigned long long>(t));
        }
    }
    if (p.acc)
        publish_if_last(frame, static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x), p.bins, p.acc, p.hist, p.sum,
                        p.sumsq, p.ctas_per_frame, p.npx, p.mean, p.stddev);
}

/// One launch clearing the histogram slots and both per-frame sums.
__global__ void zero_scratch_kernel(unsigned long long* hist, long long nh, unsigned long long* sum,
                                    unsigned long long* sumsq, int frames) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nh + 2LL * frames;
         i += stride) {
        if (i < nh) hist[i] = 0;
        else if (i < nh + frames) sum[i - nh] = 0;
        else sumsq[i - nh - frames] = 0;
    }
}

/// MeanStdDev finalize, one thread per frame:
///   mean = F32((sum * 1.0) / n);  sd = F32(sqrt(max((sumsq * 1.0) / n - m*m, 0.0)))
/// with m the F32-rounded mean (the reduce_stddev node reads the mean scalar).
__device__ __forceinline__ void meanstd_of(unsigned long long s1, unsigned long long s2, long long n, gvxb_value* mean,
                                           gvxb_value* sd) {
    const double dn = __ll2double_rn(n);
    const double m = static_cast<double>(
        __double2float_rn(__ddiv_rn(__dmul_rn(__ll2double_rn(static_cast<long long>(s1)), 1.0), dn)));
    if (mean) {
        mean->real = 1;
        mean->bits = __double_as_longlong(m);
    }
    if (sd) {
        const double ex2 = __ddiv_rn(__dmul_rn(__ll2double_rn(static_cast<long long>(s2)), 1.0), dn);
        const double var0 = __dsub_rn(ex2, __dmul_rn(m, m));
        const double var = var0 < 0.0 ? 0.0 : var0; // std::max(var0, 0.0)
        sd->real = 1;
        sd->bits = __double_as_longlong(static_cast<double>(__double2float_rn(__dsqrt_rn(var))));
    }
}

__global__ void meanstd_finalize_kernel(const unsigned long long* sum, const unsigned long long* sumsq, long long n,
                                        int frames, gvxb_value* mean, gvxb_value* sd) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= frames) return;
    meanstd_of(sum[f], sumsq[f], n, mean ? mean + f : nullptr, sd ? sd + f : nullptr);
}


// ======================================================= separable fast path
//
// Masks that factor as m = u v^T with non-negative integers (the binomial
// blurs of cfg3 / cfg4 do) and a power-of-two divisor run a packed-FP32
// pipeline: every lane owns 4 columns as (even, odd) float2 pairs, the
// horizontal K-tap pass reads its 4 + 2R source bytes from the TMA tile,
// the vertical pass streams rows through K push-accumulators (each new
// horizontal row adds u[i] * h into the K outputs it touches), and the
// rounding division is one FFMA2 in round-down mode:
//   q = floor((s + d/2) / d) = round_half_away(s / d)   (s >= 0, d = 2^k)
// landing as the float 1.5*2^23 + q whose low byte is q.  All sums are
// integers < 2^24 (checked on the host), so every step is exact.

constexpr int kSepThreads = 96;
constexpr int kSepTW = 4 * kSepThreads; // 384 columns: 4K / 8K / 1080p split evenly
constexpr int kSepSW = kSepTW + 32;     // tile origin x0 - 16 (16-byte aligned TMA start)
#ifndef GVX_SEP_HIST_THREADS
#define GVX_SEP_HIST_THREADS 128 // 4 warps: every byte of a (value, lane) counter word used (+2% with red increments)
#endif
/// Threads per CTA: the histogram modes may use all four counter bytes of a
/// (value, lane) word with four warps.
__host__ __device__ constexpr int sep_threads(int mode) { return mode >= 2 ? GVX_SEP_HIST_THREADS : kSepThreads; }
#ifndef GVX_SEP_TH_MAX
#define GVX_SEP_TH_MAX 48
#endif
constexpr int kSepTHMax = GVX_SEP_TH_MAX; // measured best of 32 / 48 / 64 (cfg3)
#ifndef GVX_SEP_HIST_TH
#define GVX_SEP_HIST_TH 40 // 4 CTAs / SM with 4-warp tiles
#endif
constexpr int kSepHistTH = GVX_SEP_HIST_TH; // u8 counters: 4 px * rows <= 255; measured best (24..60): 4 CTAs / SM
// each warp owns one byte of a (value, lane) counter word: at most 4 warps,
// and a tile's 4 px x kSepHistTH rows per lane must not carry out of a byte
static_assert(GVX_SEP_HIST_THREADS % 32 == 0 && GVX_SEP_HIST_THREADS <= 128, "one counter byte per warp");
static_assert(4 * kSepHistTH <= 255, "u8 histogram counters would wrap");
constexpr int kSepHistBytes = 256 * 32 * 4;

struct SepParams {
    int width;
    Band band;
    int th;
    int pdl_wait; // the previous grid on the stream may have written what this one touches
    float u[7], v[7];
    float bias;     // d / 2 (0 for d == 1); fractional form: (d / 2) / 2^15
    float inv_d;    // 1 / (d << shift), exact power of two
    float qscale;   // quotient FMA: 1.5*2^23 + q = rd(acc * qscale + qbase)
    float qbase;    //   magic form: inv_d, 1.5*2^23; fractional: 2^15 inv_d, 1.5*2^23 - 2^15 W inv_d
    int frac;       // 0 magic-form columns; 1 fractional form; 2 fractional + symmetric unit-end row mask
    int clamp255;   // q may exceed 255: 1 saturate to 255, 2 wrap (low byte)
    uint8_t* dst;   // K3 output, or K4's converted image (may be null)
    int64_t dst_pitch, dst_fstride;
    // K4
    gvxb_value* hist;
    int bins;
    long long offset, range;
    int identity;
    unsigned long long* sum;
    unsigned long long* sumsq;
    // one-launch form (acc != null): histogram accumulators and a CTA-done
    // counter per frame, zero on entry; the frame's last CTA publishes the
    // histogram and MeanStdDev and leaves the scratch zero again
    unsigned long long* acc; // frames x (bins + 1): bins accumulators, then the counter
    int ctas_per_frame;
    long long npx;           // pixels per frame
    gvxb_value* mean;
    gvxb_value* stddev;
};

/// Columns c+j, j = -R .. R+3, of one tile row as pairs P(j) = (c+j, c+j+2).
template <int R>
struct SepRow {
    float2 p[2 * R + 2];
};

template <int R>
__device__ __forceinline__ SepRow<R> sep_load(const uint8_t* row, int off) {
    const uint32_t wl = lds32(row, off - 4), wc = lds32(row, off), wr = lds32(row, off + 4);
    // column c + j for j = -4 .. 7 lives in byte (j & 3) of word (j >> 2) + 1
    auto col = [&](int j) -> float {
        const uint32_t w = j < 0 ? wl : (j < 4 ? wc : wr);
        return magic_byte(w, j & 3);
    };
    const float2 magic = f2(-8388608.f, -8388608.f);
    SepRow<R> r;
    // de-magic half of the pairs; the others are recombined halves
#pragma unroll
    for (int j = -R; j <= R + 1; ++j) {
        const int k = j + R;
        if ((k & 2) == 0) r.p[k] = add2(f2(col(j), col(j + 2)), magic);
    }
#pragma unroll
    for (int j = -R; j <= R + 1; ++j) {
        const int k = j + R;
        if ((k & 2) != 0) {
            // P(j) = (c+j, c+j+2) = (P(j-2).y, P(j+2).x) when both exist
            if (k - 2 >= 0 && k + 2 <= 2 * R + 1) r.p[k] = f2(r.p[k - 2].y, r.p[k + 2].x);
            else r.p[k] = add2(f2(col(j), col(j + 2)), magic);
        }
    }
    return r;
}

/// As sep_load, with every column in fractional form 1 + x / 2^15 (byte
/// permutes only, no de-biasing adds): weighted sums W + s / 2^15 stay exact
/// while W (2^15 + 255) < 2^24 (checked on the host).
template <int R, bool kHalf = false>
__device__ __forceinline__ SepRow<R> sep_load_frac(const uint8_t* row, int off) {
    const uint32_t wl = lds32(row, off - 4), wc = lds32(row, off), wr = lds32(row, off + 4);
    // kHalf: 1 + (x + 1/2) / 2^15 (bit 7 of the constant), the rounding bias
    // riding in the sources (see sep_kernel kLoad 3)
    constexpr uint32_t kBase = kHalf ? 0x3F800080u : 0x3F800000u;
    auto col = [&](int j) -> float {
        const uint32_t w = j < 0 ? wl : (j < 4 ? wc : wr);
        return __uint_as_float(__byte_perm(w, kBase, 0x7604u | (static_cast<unsigned>(j & 3) << 4)));
    };
    SepRow<R> r;
#pragma unroll
    for (int j = -R; j <= R + 1; ++j) r.p[j + R] = f2(col(j), col(j + 2));
    return r;
}

/// Horizontal pass of a symmetric row mask with unit ends (v[t] = v[K-1-t],
/// v[0] = 1: the binomials): outer pairs added first, K - 1 instead of K
/// packed ops per column pair.
template <int K>
__device__ __forceinline__ Q4 sep_horizontal_sym(const SepRow<K / 2>& r, const float* v) {
    constexpr int R = K / 2;
    Q4 h{add2(r.p[0], r.p[K - 1]), add2(r.p[1], r.p[K])};
#pragma unroll
    for (int t = 1; t < R; ++t) {
        h.e = fma2(f2(v[t], v[t]), add2(r.p[t], r.p[K - 1 - t]), h.e);
        h.o = fma2(f2(v[t], v[t]), add2(r.p[t + 1], r.p[K - t]), h.o);
    }
    h.e = fma2(f2(v[R], v[R]), r.p[R], h.e);
    h.o = fma2(f2(v[R], v[R]), r.p[R + 1], h.o);
    return h;
}

template <int K>
__device__ __forceinline__ Q4 sep_horizontal(const SepRow<K / 2>& r, const float* v) {
    Q4 h;
    h.e = mul2(f2(v[0], v[0]), r.p[0]);
    h.o = mul2(f2(v[0], v[0]), r.p[1]);
#pragma unroll
    for (int t = 1; t < K; ++t) {
        h.e = fma2(f2(v[t], v[t]), r.p[t], h.e);
        h.o = fma2(f2(v[t], v[t]), r.p[t + 1], h.o);
    }
    return h;
}

/// Division epilogue: 1.5*2^23 + min(q, 255) per column.
__device__ __forceinline__ Q4 sep_quotient(Q4 acc, float qscale, float qbase, int clamp255) {
    const float2 M = f2(qbase, qbase), id = f2(qscale, qscale);
    Q4 q{__ffma2_rd(acc.e, id, M), __ffma2_rd(acc.o, id, M)};
    if (clamp255) {
        const float top = 12582912.f + 255.f;
        q.e = f2(fminf(q.e.x, top), fminf(q.e.y, top));
        q.o = f2(fminf(q.o.x, top), fminf(q.o.y, top));
    }
    return q;
}

__device__ __forceinline__ Q4 sep_neg_quotient(Q4 acc, float qscale, float qbase, int clamp255) {
    const float2 M = f2(-qbase, -qbase), id = f2(-qscale, -qscale);
    Q4 q{__ffma2_ru(acc.e, id, M), __ffma2_ru(acc.o, id, M)};
    if (clamp255) {
        const float bot = -12582912.f - 255.f;
        q.e = f2(fmaxf(q.e.x, bot), fmaxf(q.e.y, bot));
        q.o = f2(fmaxf(q.o.x, bot), fmaxf(q.o.y, bot));
    }
    return q;
}

/// Counter increment as one shared-memory reduction on the (value, lane)
/// word: each warp owns one byte of it (inc = 1 << 8 warp), at most
/// 4 px x kSepHistTH rows counts per byte between merges (static_assert
/// below), so no carry crosses bytes.  No load -> add -> store dependency
/// chain per pixel.
__device__ __forceinline__ void smem_red_u32(uint32_t addr, uint32_t inc) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(inc) : "memory");
}

/// ++ of a u8 shared-memory counter.  Volatile asm keeps the increments of
/// one thread in program order (two may hit the same counter) while leaving
/// the tile loads free to be scheduled around them.
__device__ __forceinline__ void smem_inc_u8(uint32_t addr) {
    asm volatile(
        "{\n"
        ".reg .u16 t;\n"
        "ld.shared.u8 t, [%0];\n"
        "add.u16 t, t, 1;\n"
        "st.shared.u8 [%0], t;\n"
        "}\n" ::"r"(addr));
}

/// Low bytes of (e.x, o.x, e.y, o.y) = columns c .. c+3.
__device__ __forceinline__ uint32_t sep_pack(Q4 q) {
    const uint32_t a = __byte_perm(__float_as_uint(q.e.x), __float_as_uint(q.o.x), 0x0040u);
    const uint32_t b = __byte_perm(__float_as_uint(q.e.y), __float_as_uint(q.o.y), 0x0040u);
    return __byte_perm(a, b, 0x5410u);
}

__device__ __forceinline__ void store4(uint8_t* dp, uint32_t w, int c, int width) {
    if (c + 3 < width) {
        *reinterpret_cast<uint32_t*>(dp) = w;
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (c + i < width) dp[i] = static_cast<uint8_t>(w >> (8 * i));
    }
}

/// kMode 0: U8 stencil output; 1: unsharp chain sat_u8(2x - blur);
/// 2: Convolve -> ConvertDepth -> per-CTA value histogram; 3: as 2 and also
/// store the converted image.
template <int K, int kMode, bool kClamp, int kLoad, bool kPub = false>
__global__ void __launch_bounds__(sep_threads(kMode)) sep_kernel(const __grid_constant__ CUtensorMap map, SepParams p) {
    constexpr int NT = sep_threads(kMode), TW = 4 * NT, SW = TW + 32;
    constexpr int R = K / 2;
    constexpr int SH = (kMode >= 2 ? kSepHistTH : kSepTHMax) + 2 * R;
    __shared__ alignas(128) uint8_t tile[SH * SW];
    __shared__ uint64_t bar;
    extern __shared__ uint4 hist_dyn[]; // kMode 2: [bin][lane][warp] u8 counters
    uint8_t* hist = reinterpret_cast<uint8_t*>(hist_dyn);
    const int tid = static_cast<int>(threadIdx.x);
    if (kMode >= 2) { // shared memory only: may overlap the previous grid's tail
        for (int i = tid; i < kSepHistBytes / 16; i += NT) hist_dyn[i] = make_uint4(0, 0, 0, 0);
    }
    pdl_prologue(p.pdl_wait);

    const int x0 = blockIdx.x * TW;
    const int y0 = p.band.row0 + blockIdx.y * p.th;
    const int n = min(y0 + p.th, p.band.row1) - y0;
    const int frame = blockIdx.z;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    stage_tile_u8<SW, SH>(tile, &map, &bar, x0 - 16, y0 - R, frame, p.width, p.band, p.th + 2 * R);

    const int c = x0 + 4 * tid;
    const int off = 16 + 4 * tid;
    const int dy0 = kMode >= 2 ? y0 : y0 - p.band.dst_row0;
    uint8_t* drow = p.dst ? p.dst + frame * p.dst_fstride + static_cast<int64_t>(dy0) * p.dst_pitch + c : nullptr;
    const uint8_t* crow = tile + R * SW + off; // kMode 1: centre pixels of output row o
    // kMode 2 counter of (value, lane, warp): value * 128 + lane * 4 + warp
    const uint32_t hbase = smem_u32(hist_dyn) + (((tid & 31) << 2) | (tid >> 5));
    const uint32_t hcnt = hbase - (0x4B400000u << 7);
    const uint32_t hword = smem_u32(hist_dyn) + ((tid & 31) << 2); // the (value 0, lane) word
    const uint32_t hwcnt = hword - (0x4B400000u << 7);
    const uint32_t hinc = 1u << (8 * (tid >> 5));                  // this warp's byte
    float u[K], v[K];
#pragma unroll
    for (int t = 0; t < K; ++t) u[t] = p.u[t], v[t] = p.v[t];
    const float2 bias = f2(p.bias, p.bias);

    // kEdge: this strip crosses the right image border, so lanes may own
    // fewer than 4 (or no) columns; interior strips run without any checks
    auto body = [&](auto edge_tag) {
        constexpr bool kEdge = decltype(edge_tag)::value;
        const bool live = !kEdge || c < p.width, full = !kEdge || c + 3 < p.width;
        const int nv = kEdge ? min(4, p.width - c) : 4;
        auto store = [&](uint32_t w) {
            if (full) {
                *reinterpret_cast<uint32_t*>(drow) = w;
            } else if (live) {
                for (int i = 0; i < nv; ++i) drow[i] = static_cast<uint8_t>(w >> (8 * i));
            }
        };
        // qv = 1.5*2^23 + value has bits 0x4B400000 + value, so one
        // multiply-add gives the counter address hbase + value * 128
        auto count = [&](float qv, int i) {
            if (kEdge && i >= nv) return;
#ifdef GVX_SEP_HIST_LDST
            if (kClamp && p.clamp255 == 2) smem_inc_u8(hbase + ((__float_as_uint(qv) & 0xFFu) << 7)); // Wrap
            else smem_inc_u8(hcnt + (__float_as_uint(qv) << 7));
#else
            if (kClamp && p.clamp255 == 2) smem_red_u32(hword + ((__float_as_uint(qv) & 0xFFu) << 7), hinc); // Wrap
            else smem_red_u32(hwcnt + (__float_as_uint(qv) << 7), hinc);
#endif
        };
        Q4 pend{};
        bool have_pend = false;
        auto emit = [&](Q4 acc) {
            if (kMode == 1) {
#ifndef GVX_SEP_FMNMX_CLAMP
                // -(1.5*2^23 + b) by round-up of the negated product; the centre
                // pixels as 1.5*2^23 + x, so 2(1.5*2^23 + x) - (1.5*2^23 + b) =
                // 1.5*2^23 + y, y = 2x - b in [-255, 510], whose low 16 bits are
                // y (two's complement); the U8 saturation runs as s16x2 max / min
                // on two columns per register
                const Q4 q = sep_neg_quotient(acc, p.qscale, p.qbase, kClamp);
                const uint32_t w = *reinterpret_cast<const uint32_t*>(crow);
                auto centre = [&](int k) { return __uint_as_float(__byte_perm(w, 0x4B400000u, 0x7640u | k)); };
                const float2 two = f2(2.f, 2.f);
                const float2 ue = fma2(two, f2(centre(0), centre(2)), q.e), uo = fma2(two, f2(centre(1), centre(3)), q.o);
                uint32_t lo = __byte_perm(__float_as_uint(ue.x), __float_as_uint(uo.x), 0x5410u); // columns c, c+1
                uint32_t hi = __byte_perm(__float_as_uint(ue.y), __float_as_uint(uo.y), 0x5410u); // columns c+2, c+3
                asm("max.s16x2 %0, %0, %1;" : "+r"(lo) : "r"(0u));
                asm("max.s16x2 %0, %0, %1;" : "+r"(hi) : "r"(0u));
                asm("min.s16x2 %0, %0, %1;" : "+r"(lo) : "r"(0x00FF00FFu));
                asm("min.s16x2 %0, %0, %1;" : "+r"(hi) : "r"(0x00FF00FFu));
                store(__byte_perm(lo, hi, 0x6420u));
#else
                // -(1.5*2^23 + b) by round-up of the negated product, then
                // 2(2^23 + x) - (1.5*2^23 + b) = 2^22 + (2x - b), clamped to U8
                const Q4 q = sep_neg_quotient(acc, p.qscale, p.qbase, kClamp);
                const uint32_t w = *reinterpret_cast<const uint32_t*>(crow);
                const float2 xe = f2(magic_byte(w, 0), magic_byte(w, 2)), xo = f2(magic_byte(w, 1), magic_byte(w, 3));
                const float2 two = f2(2.f, 2.f), lift = f2(8388608.f, 8388608.f);
                float2 re = fma2(two, xe, q.e), ro = fma2(two, xo, q.o);
                const float lo = 4194304.f, hi = 4194304.f + 255.f;
                re = f2(fminf(fmaxf(re.x, lo), hi), fminf(fmaxf(re.y, lo), hi));
                ro = f2(fminf(fmaxf(ro.x, lo), hi), fminf(fmaxf(ro.y, lo), hi));
                store(sep_pack(Q4{add2(re, lift), add2(ro, lift)})); // 1.5*2^23 + y
#endif
                crow += SW;
                drow += p.dst_pitch;
            } else if (kMode == 0) {
                store(sep_pack(sep_quotient(acc, p.qscale, p.qbase, kClamp)));
                drow += p.dst_pitch;
            } else {
                const Q4 q = sep_quotient(acc, p.qscale, p.qbase, kClamp && p.clamp255 == 1);
                if (kMode == 3) {
                    store(sep_pack(q));
                    drow += p.dst_pitch;
                }
                // count the PREVIOUS row now: its increment chain overlaps
                // this row's arithmetic instead of ending it
                if (have_pend) {
                    count(pend.e.x, 0);
                    count(pend.o.x, 1);
                    count(pend.e.y, 2);
                    count(pend.o.y, 3);
                }
                pend = q;
                have_pend = true;
            }
        };
        // push accumulation: smem row j (global row y0 - R + j) adds u[i] * h(j)
        // into output o = j - i; output o is complete after row j = o + K - 1.
        Q4 acc[K];
        Q4 hq[K]; // kLoad 3: the last K rows' horizontal sums (slot = row mod K)
        auto row = [&](int j, int slot0) { // slot0 = j mod K
            // kLoad 0: magic form; 1: fractional form; 2: fractional + symmetric
            // row mask; 3: as 2 with symmetric column mask and the rounding
            // bias in the sources: rows kept, outputs summed symmetrically
            const Q4 h = kLoad == 3 ? sep_horizontal_sym<K>(sep_load_frac<R, true>(tile + j * SW, off), v)
                         : kLoad == 2 ? sep_horizontal_sym<K>(sep_load_frac<R>(tile + j * SW, off), v)
                                      : sep_horizontal<K>(kLoad == 1 ? sep_load_frac<R>(tile + j * SW, off)
                                                                     : sep_load<R>(tile + j * SW, off),
                                                          v);
            if constexpr (kLoad == 3) {
                hq[slot0] = h;
                return;
            }
#pragma unroll
            for (int i = 0; i < K; ++i) {
                Q4& a = acc[(slot0 - i + 2 * K) % K];
                if (i == 0) a = Q4{fma2(f2(u[0], u[0]), h.e, bias), fma2(f2(u[0], u[0]), h.o, bias)};
                else a = Q4{fma2(f2(u[i], u[i]), h.e, a.e), fma2(f2(u[i], u[i]), h.o, a.o)};
            }
        };
        /// kLoad 3: output o from rows o .. o+K-1 (row o+K-1 in slot `last`):
        /// (h0 + h_{K-1}) + sum u_i (h_i + h_{K-1-i}) + u_R h_R.
        auto vsum = [&](int last) {
            auto at = [&](int i) -> const Q4& { return hq[(last + 1 + i) % K]; };
            Q4 a{add2(at(0).e, at(K - 1).e), add2(at(0).o, at(K - 1).o)};
#pragma unroll
            for (int i = 1; i < R; ++i) {
                a.e = fma2(f2(u[i], u[i]), add2(at(i).e, at(K - 1 - i).e), a.e);
                a.o = fma2(f2(u[i], u[i]), add2(at(i).o, at(K - 1 - i).o), a.o);
            }
            a.e = fma2(f2(u[R], u[R]), at(R).e, a.e);
            a.o = fma2(f2(u[R], u[R]), at(R).o, a.o);
            return a;
        };
#pragma unroll
        for (int j = 0; j < K - 1; ++j) row(j, j);
        auto block = [&](int O, auto checked) { // K output rows O .. O+K-1 (O a multiple of K)
#pragma unroll
            for (int t = 0; t < K; ++t) {
                if (decltype(checked)::value && O + t >= n) break;
                row(O + t + K - 1, (t + K - 1) % K);
                if constexpr (kLoad == 3) emit(vsum((t + K - 1) % K));
                else emit(acc[t]); // output o = O + t
            }
        };
        int O = 0;
        for (; O + K <= n; O += K) block(O, std::false_type{}); // whole blocks: no row checks
        if (O < n) block(O, std::true_type{});
        if (kMode >= 2 && have_pend) {
            count(pend.e.x, 0);
            count(pend.o.x, 1);
            count(pend.e.y, 2);
            count(pend.o.y, 3);
        }
    };
    if (x0 + TW > p.width) body(std::true_type{});
    else body(std::false_type{});

    if (kMode < 2) return;
    __syncthreads();
    // merge: thread t owns values t, t + NT, ... (< 256); the 128 counter
    // bytes of a value are read as 8 uint4 in a rotated order (bank spread)
    long long s1 = 0, s2 = 0;
    for (int val = tid; val < 256; val += NT) {
        const uint4* rowp = hist_dyn + val * 8;
        unsigned cnt = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint4 q = rowp[(k + val) & 7];
            cnt = __dp4a(q.x, 0x01010101u, cnt);
            cnt = __dp4a(q.y, 0x01010101u, cnt);
            cnt = __dp4a(q.z, 0x01010101u, cnt);
            cnt = __dp4a(q.w, 0x01010101u, cnt);
        }
        if (!cnt) continue;
        s1 += static_cast<long long>(cnt) * val;
        s2 += static_cast<long long>(cnt) * val * val;
        if (p.hist) {
            long long bin = val;
            if (!p.identity) {
                const long long t = (static_cast<long long>(val) - p.offset) * p.bins;
                bin = t / p.range;
            }
            if (bin < 0 || bin >= p.bins) continue; // out of range: skipped (ref:src/execute.cpp:717-724)
            unsigned long long* slot =
                kPub ? p.acc + static_cast<int64_t>(frame) * (p.bins + 1) + bin
                     : reinterpret_cast<unsigned long long*>(&p.hist[static_cast<int64_t>(frame) * p.bins + bin].bits);
            atomicAdd(slot, static_cast<unsigned long long>(cnt));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((tid & 31) == 0) {
        atomicAdd(&p.sum[frame], static_cast<unsigned long long>(s1));
        atomicAdd(&p.sumsq[frame], static_cast<unsigned long long>(s2));
    }
    // the one-launch form is its own instantiation: a (skipped) epilogue in
    // the batch kernel cost it 2.4% (measured)
    if constexpr (kPub)
        publish_if_last(frame, tid, NT, p.bins, p.acc, p.hist, p.sum, p.sumsq, p.ctas_per_frame, p.npx, p.mean,
                        p.stddev);
}

} // namespace gvxd

using namespace gvxd;

namespace {

/// m = u v^T with non-negative integer u, v (v primitive).
bool factor_mask(const int32_t* m, int K, int* u, int* v) {
    int i0 = -1, j0 = -1;
    for (int i = 0; i < K * K; ++i) {
        if (m[i] < 0) return false;
        if (m[i] && i0 < 0) i0 = i / K, j0 = i % K;
    }
    if (i0 < 0) return false;
    long long g = 0;
    for (int j = 0; j < K; ++j) {
        long long a = m[i0 * K + j], b = g;
        while (b) { long long t = a % b; a = b; b = t; }
        g = a;
    }
    for (int j = 0; j < K; ++j) v[j] = static_cast<int>(m[i0 * K + j] / g);
    for (int i = 0; i < K; ++i) {
        if (m[i * K + j0] % v[j0]) return false;
        u[i] = m[i * K + j0] / v[j0];
        for (int j = 0; j < K; ++j)
            if (static_cast<long long>(u[i]) * v[j] != m[i * K + j]) return false;
    }
    return true;
}

bool is_pow2(long long d) { return d >= 1 && (d & (d - 1)) == 0; }

/// Fills the separable parameters when the fast path is exact for this
/// mask / divisor; returns the largest quotient floor((255 sum + d/2) / d).
bool sep_setup(const int32_t* mask, int K, long long d, int shift, SepParams& p, long long& qmax) {
    int u[7], v[7];
    if (!is_pow2(d) || shift < 0 || shift > 16 || !factor_mask(mask, K, u, v)) return false;
    long long su = 0, sv = 0;
    for (int t = 0; t < K; ++t) su += u[t], sv += v[t];
    const long long smax = 255 * su * sv + d / 2;
    if (255 * sv >= (1 << 24) || smax >= (1 << 24)) return false;
    for (int t = 0; t < 7; ++t) p.u[t] = t < K ? static_cast<float>(u[t]) : 0.f, p.v[t] = t < K ? static_cast<float>(v[t]) : 0.f;
    p.bias = static_cast<float>(d / 2);
    p.inv_d = 1.0f / static_cast<float>(d << shift);
    p.qscale = p.inv_d;
    p.qbase = 12582912.f;
    // fractional form (columns as 1 + x / 2^15, no de-biasing adds): exact
    // while W (2^15 + 255) + d/2 < 2^24 and 2^15 W / (d << shift) is an integer
    const long long W = su * sv, D = d << shift;
    p.frac = W * (32768 + 255) + d / 2 < (1LL << 24) && (W * 32768) % D == 0 ? 1 : 0;
    if (std::getenv("GVX_SEP_NOFRAC")) p.frac = 0; // A/B tests
    bool sym = v[0] == 1 && !std::getenv("GVX_SEP_NOSYM");
    for (int t = 0; t < K; ++t) sym = sym && v[t] == v[K - 1 - t];
    if (p.frac && sym) p.frac = 2;
    // both masks symmetric with unit ends, even sums and d == W: the bias d/2
    // = W/2 rides in the sources as +1/2 each, so no output needs a bias add
    // and every partial sum stays a multiple of 2^-15 (exact)
    bool usym = u[0] == 1 && su % 2 == 0 && sv % 2 == 0 && W == d && !std::getenv("GVX_SEP_NOVSYM");
    for (int t = 0; t < K; ++t) usym = usym && u[t] == u[K - 1 - t];
    if (p.frac == 2 && usym) p.frac = 3;
    if (p.frac) {
        p.bias = p.frac == 3 ? 0.f : static_cast<float>(d / 2) / 32768.f;
        p.qscale = 32768.f / static_cast<float>(D);
        p.qbase = static_cast<float>(12582912LL - W * 32768 / D);
    }
    qmax = smax / d;
    return true;
}

template <int K, int M, int F>
void* sep_fn(bool clamp) {
    return clamp ? reinterpret_cast<void*>(&sep_kernel<K, M, true, F>)
                 : reinterpret_cast<void*>(&sep_kernel<K, M, false, F>);
}

template <int K, int M>
void* sep_fn_f(bool clamp, int frac) {
    switch (frac) {
    case 3: return sep_fn<K, M, 3>(clamp);
    case 2: return sep_fn<K, M, 2>(clamp);
    case 1: return sep_fn<K, M, 1>(clamp);
    default: return sep_fn<K, M, 0>(clamp);
    }
}

/// The one-launch (publishing) conv+stats kernels: modes 2 / 3 with the
/// fractional-symmetric load (the binomial masks); others run the batch form.
template <int M>
void* sep_fn_pub(int k, bool clamp, int frac) {
    if (frac != 3) return nullptr;
    switch (k) {
    case 3: return clamp ? reinterpret_cast<void*>(&sep_kernel<3, M, true, 3, true>)
                         : reinterpret_cast<void*>(&sep_kernel<3, M, false, 3, true>);
    case 5: return clamp ? reinterpret_cast<void*>(&sep_kernel<5, M, true, 3, true>)
                         : reinterpret_cast<void*>(&sep_kernel<5, M, false, 3, true>);
    case 7: return clamp ? reinterpret_cast<void*>(&sep_kernel<7, M, true, 3, true>)
                         : reinterpret_cast<void*>(&sep_kernel<7, M, false, 3, true>);
    default: return nullptr;
    }
}

template <int M>
void* sep_fn_k(int k, bool clamp, int frac) {
    switch (k) {
    case 3: return sep_fn_f<3, M>(clamp, frac);
    case 5: return sep_fn_f<5, M>(clamp, frac);
    case 7: return sep_fn_f<7, M>(clamp, frac);
    default: return nullptr;
    }
}

int sep_launch(gvxb_ctx ctx, void* fn, const gvxb_image& s, SepParams& p, int K, int rows, int th_max, size_t dyn,
               int ch_threads, const gvxb_range* wr, int nw, const gvxb_range* rd = nullptr) {
    using namespace gvxb_impl;
    if (dyn > 0) { // static tile + dynamic histogram exceed the 48 KB default
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
        if (e != cudaSuccess) return cuda_fail(e, "separable stencil smem attribute");
    }
    int per_sm = 0;
    const int nt = ch_threads;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, dyn);
    const int frames = s.frames > 0 ? s.frames : 1;
    const int tw = 4 * nt, sw = tw + 32;
    const long long strips = static_cast<long long>((s.width + tw - 1) / tw) * frames;
    p.th = balanced_tile_rows(strips, rows, static_cast<long long>(per_sm > 0 ? per_sm : 1) * ctx->sm_count, th_max,
                              K - 1);
    if (const char* e = std::getenv("GVX_SEP_TH")) p.th = std::max(8, std::min(th_max, std::atoi(e))); // tuning experiments
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, sw, p.th + K - 1)) return rc;
    dim3 grid((s.width + tw - 1) / tw, (rows + p.th - 1) / p.th, frames);
    if (p.acc) p.ctas_per_frame = static_cast<int>(grid.x * grid.y);
    const gvxb_range r[1] = {rd ? *rd : image_range(s)};
    p.pdl_wait = pdl_must_wait(ctx, r, 1, wr, nw);
    void* args[] = {&map, &p};
    return launch_tracked(ctx, fn, grid, dim3(nt), args, dyn, r, 1, wr, nw, "separable stencil kernel");
}

template <int K>
void* stencil_fn(int mode) {
    return mode == 0 ? reinterpret_cast<void*>(&stencil_point_kernel<K, 0>)
                     : reinterpret_cast<void*>(&stencil_point_kernel<K, 1>);
}

void range_of(int fmt, int& lo, int& hi) {
    switch (fmt) {
    case GVXB_U8: lo = 0, hi = 255; break;
    case GVXB_S16: lo = -32768, hi = 32767; break;
    case GVXB_U16: lo = 0, hi = 65535; break;
    default: lo = INT32_MIN, hi = INT32_MAX; break;
    }
}

} // namespace

extern "C" int gvxb_stencil_point(gvxb_ctx ctx, const gvxb_stencil_args* a) {
    using namespace gvxb_impl;
    const gvxb_image& s = a->src;
    if (s.format != GVXB_U8 || a->dst.format != GVXB_U8) return fail(GVXB_ERR_INVALID, "stencil: U8 -> U8 only");
    if (a->div_num != 1 || a->div_den < 1) return fail(GVXB_ERR_INVALID, "stencil: divisor must be 1/d");
    const int rows = a->band.row1 - a->band.row0;
    if (rows <= 0 || s.width <= 0) return GVXB_OK;
    if (a->mode == 0 || a->mode == 1) {
        SepParams sp{};
        long long qmax = 0;
        if (sep_setup(a->mask, a->ksize, a->div_den, 0, sp, qmax)) {
            sp.width = s.width;
            sp.band = Band{a->band.row0, a->band.row1, a->band.global_h, a->band.src_row0, a->band.dst_row0};
            sp.clamp255 = qmax > 255;
            sp.dst = static_cast<uint8_t*>(a->dst.data);
            sp.dst_pitch = a->dst.pitch;
            sp.dst_fstride = a->dst.frames > 1 ? a->dst.frame_stride : a->dst.pitch * a->dst.height;
            void* fn = a->mode == 0 ? sep_fn_k<0>(a->ksize, sp.clamp255, sp.frac) : sep_fn_k<1>(a->ksize, sp.clamp255, sp.frac);
            // the band's rows (plus the K/2 halo read above and below) only, so
            // launches on disjoint row bands of one buffer stay independent
            const int b0 = a->band.row0, hk = a->ksize / 2;
            const gvxb_range rd = rows_range(s, b0 - hk - a->band.src_row0, rows + 2 * hk);
            const gvxb_range w[1] = {rows_range(a->dst, b0 - a->band.dst_row0, rows)};
            if (fn) return sep_launch(ctx, fn, s, sp, a->ksize, rows, kSepTHMax, 0, sep_threads(0), w, 1, &rd);
        }
    }
    StencilParams p;
    p.width = s.width;
    p.band = Band{a->band.row0, a->band.row1, a->band.global_h, a->band.src_row0, a->band.dst_row0};
    for (int i = 0; i < 49; ++i) p.mask[i] = a->mask[i];
    p.div = static_cast<int>(a->div_den);
    range_of(GVXB_U8, p.out_lo, p.out_hi);
    p.mode = a->mode;
    p.dst = static_cast<uint8_t*>(a->dst.data);
    p.dst_pitch = a->dst.pitch;
    p.dst_fstride = a->dst.frames > 1 ? a->dst.frame_stride : a->dst.pitch * a->dst.height;
    void* fn = nullptr;
    int sh = 0;
    switch (a->ksize) {
    case 3: fn = stencil_fn<3>(a->mode), sh = kStTH + 2; break;
    case 5: fn = stencil_fn<5>(a->mode), sh = kStTH + 4; break;
    case 7: fn = stencil_fn<7>(a->mode), sh = kStTH + 6; break;
    default: return fail(GVXB_ERR_UNSUPPORTED, "stencil: ksize must be 3, 5 or 7");
    }
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, kStSW, sh)) return rc;
    const int frames = s.frames > 0 ? s.frames : 1;
    dim3 grid((s.width + kStTW - 1) / kStTW, (rows + kStTH - 1) / kStTH, frames);
    void* args[] = {&map, &p};
    untracked_op(ctx);
    cudaError_t e = cudaLaunchKernel(fn, grid, dim3(kStThreads), args, 0, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "stencil kernel launch");
    return check_launch(ctx, "stencil kernel");
}

static int meanstd(gvxb_ctx ctx, const gvxb_conv_stats_args* a, const ConvStatsParams& p, int frames, const gvxb_image& s) {
    if (a->mean || a->stddev) {
        const long long n = static_cast<long long>(s.width) * s.height;
        gvxb_impl::untracked_op(ctx);
        meanstd_finalize_kernel<<<(frames + 63) / 64, 64, 0, ctx->stream>>>(p.sum, p.sumsq, n, frames, a->mean,
                                                                              a->stddev);
        return gvxb_impl::check_launch(ctx, "meanstd finalize");
    }
    return GVXB_OK;
}

extern "C" int gvxb_conv_stats(gvxb_ctx ctx, const gvxb_conv_stats_args* a) {
    using namespace gvxb_impl;
    const gvxb_image& s = a->src;
    if (s.format != GVXB_U8) return fail(GVXB_ERR_INVALID, "conv_stats: source must be U8");
    if (!a->sum || !a->sumsq) return fail(GVXB_ERR_INVALID, "conv_stats: sum scratch required");
    if (a->scale < 1) return fail(GVXB_ERR_INVALID, "conv_stats: scale must be >= 1");
    const int frames = s.frames > 0 ? s.frames : 1;
    ConvStatsParams p{};
    p.width = s.width;
    p.height = s.height;
    p.band = Band{0, s.height, s.height, 0, 0};
    for (int i = 0; i < 49; ++i) p.mask[i] = a->mask[i];
    p.div = static_cast<int>(a->scale);
    range_of(a->conv_format, p.conv_lo, p.conv_hi);
    p.shift = a->shift;
    p.wrap = a->wrap;
    p.bins = a->bins > 0 ? a->bins : 1;
    p.offset = a->offset;
    p.range = a->range;
    p.identity_bins = (a->offset == 0 && a->bins == a->range) ? 1 : 0;
    p.conv_out = static_cast<uint8_t*>(a->converted.data);
    p.conv_pitch = a->converted.pitch;
    p.conv_fstride = a->converted.frames > 1 ? a->converted.frame_stride : a->converted.pitch * a->converted.height;
    p.hist = a->hist;
    p.sum = reinterpret_cast<unsigned long long*>(a->sum);
    p.sumsq = reinterpret_cast<unsigned long long*>(a->sumsq);
    if (a->range == 0 && !p.identity_bins) return fail(GVXB_ERR_DIV_BY_ZERO, "histogram range is zero");

    auto clear_scratch = [&]() -> int {
        const long long nh = a->hist ? static_cast<long long>(frames) * p.bins * 2 : 0;
        const long long total = nh + 2LL * frames;
        const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 1024));
        untracked_op(ctx);
        zero_scratch_kernel<<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<unsigned long long*>(a->hist), nh,
                                                             p.sum, p.sumsq, frames);
        return check_launch(ctx, "conv_stats scratch clear");
    };
    cudaError_t e = cudaSuccess;

    {
        SepParams sp{};
        long long qmax = 0;
        int lo = 0, hi = 0;
        range_of(a->conv_format, lo, hi);
        if (sep_setup(a->mask, a->ksize, a->scale, a->shift, sp, qmax) && qmax <= hi && sep_fn_k<2>(a->ksize, false, 0)) {
            sp.width = s.width;
            sp.band = Band{0, s.height, s.height, 0, 0};
            sp.clamp255 = (qmax >> a->shift) > 255 ? (a->wrap ? 2 : 1) : 0;
            sp.dst = static_cast<uint8_t*>(a->converted.data);
            sp.dst_pitch = a->converted.pitch;
            sp.dst_fstride = p.conv_fstride;
            sp.hist = a->hist;
            sp.bins = p.bins;
            sp.offset = a->offset;
            sp.range = a->range;
            sp.identity = p.identity_bins;
            sp.sum = p.sum;
            sp.sumsq = p.sumsq;
            void* fn = sp.dst ? sep_fn_k<3>(a->ksize, sp.clamp255, sp.frac) : sep_fn_k<2>(a->ksize, sp.clamp255, sp.frac);
            void* pub = sp.dst ? sep_fn_pub<3>(a->ksize, sp.clamp255, sp.frac) : sep_fn_pub<2>(a->ksize, sp.clamp255, sp.frac);
            if (a->work && frames == 1 && pub) {
                // one launch (single frames: one execution per call; a batch
                // amortises the clear / finalize launches and would pay the
                // end-of-CTA fence in every CTA instead, measured -7% at 64
                // frames): the frame's last CTA publishes histogram and statistics
                // and re-zeroes the scratch; every written range is tracked, so the
                // next execution waits for this one after its prologue (the
                // shared-memory histogram clear overlaps this grid's tail)
                sp.acc = reinterpret_cast<unsigned long long*>(a->work);
                sp.npx = static_cast<long long>(s.width) * s.height;
                sp.mean = a->mean;
                sp.stddev = a->stddev;
                const size_t fb = static_cast<size_t>(frames) * 8;
                const gvxb_range w[5] = {image_range(a->converted), bytes_range(a->hist, 2 * fb * p.bins),
                                         bytes_range(a->work, fb * (p.bins + 1)), bytes_range(a->sum, fb),
                                         bytes_range(a->sumsq, fb)};
                return sep_launch(ctx, pub, s, sp, a->ksize, s.height, kSepHistTH, kSepHistBytes, sep_threads(2), w, 5);
            }
            if (int rc = clear_scratch()) return rc;
            const gvxb_range w[1] = {image_range(a->converted)}; // after the (untracked) scratch clear: waits anyway
            if (int rc = sep_launch(ctx, fn, s, sp, a->ksize, s.height, kSepHistTH, kSepHistBytes, sep_threads(2), w, 1))
                return rc;
            return meanstd(ctx, a, p, frames, s);
        }
    }
    void* fn = nullptr;
    int sh = 0;
    switch (a->ksize) {
    case 3: fn = reinterpret_cast<void*>(&conv_stats_kernel<3>), sh = kStTH + 2; break;
    case 5: fn = reinterpret_cast<void*>(&conv_stats_kernel<5>), sh = kStTH + 4; break;
    case 7: fn = reinterpret_cast<void*>(&conv_stats_kernel<7>), sh = kStTH + 6; break;
    default: return fail(GVXB_ERR_UNSUPPORTED, "conv_stats: ksize must be 3, 5 or 7");
    }
    dim3 grid((s.width + kStTW - 1) / kStTW, (s.height + kStTH - 1) / kStTH, frames);
    p.acc = frames == 1 ? reinterpret_cast<unsigned long long*>(a->work) : nullptr;
    if (p.acc) {
        p.ctas_per_frame = static_cast<int>(grid.x * grid.y);
        p.npx = static_cast<long long>(s.width) * s.height;
        p.mean = a->mean;
        p.stddev = a->stddev;
    } else if (int rc = clear_scratch()) {
        return rc;
    }
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, kStSW, sh)) return rc;
    const size_t dyn = sizeof(unsigned) * (kStThreads / 32) * static_cast<size_t>(p.bins);
    if (dyn > 48 * 1024) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
        if (e != cudaSuccess) return cuda_fail(e, "conv_stats smem attribute");
    }
    void* args[] = {&map, &p};
    untracked_op(ctx);
    e = cudaLaunchKernel(fn, grid, dim3(kStThreads), args, dyn, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "conv_stats kernel launch");
    if (int rc = check_launch(ctx, "conv_stats kernel")) return rc;
    return p.acc ? GVXB_OK : meanstd(ctx, a, p, frames, s);
}
