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
#include "tile.cuh"

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
};

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
            if (t)
                atomicAdd(reinterpret_cast<unsigned long long*>(&p.hist[static_cast<int64_t>(frame) * p.bins + b].bits),
                          static_cast<unsigned long long>(t));
        }
    }
}

/// MeanStdDev finalize, one thread per frame:
///   mean = F32((sum * 1.0) / n);  sd = F32(sqrt(max((sumsq * 1.0) / n - m*m, 0.0)))
/// with m the F32-rounded mean (the reduce_stddev node reads the mean scalar).
__global__ void meanstd_finalize_kernel(const unsigned long long* sum, const unsigned long long* sumsq, long long n,
                                        int frames, gvxb_value* mean, gvxb_value* sd) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= frames) return;
    const double dn = __ll2double_rn(n);
    const double m = static_cast<double>(
        __double2float_rn(__ddiv_rn(__dmul_rn(__ll2double_rn(static_cast<long long>(sum[f])), 1.0), dn)));
    if (mean) {
        mean[f].real = 1;
        mean[f].bits = __double_as_longlong(m);
    }
    if (sd) {
        const double ex2 = __ddiv_rn(__dmul_rn(__ll2double_rn(static_cast<long long>(sumsq[f])), 1.0), dn);
        const double var0 = __dsub_rn(ex2, __dmul_rn(m, m));
        const double var = var0 < 0.0 ? 0.0 : var0; // std::max(var0, 0.0)
        sd[f].real = 1;
        sd[f].bits = __double_as_longlong(static_cast<double>(__double2float_rn(__dsqrt_rn(var))));
    }
}

} // namespace gvxd

using namespace gvxd;

namespace {

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
    cudaError_t e = cudaLaunchKernel(fn, grid, dim3(kStThreads), args, 0, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "stencil kernel launch");
    return check_launch(ctx, "stencil kernel");
}

extern "C" int gvxb_conv_stats(gvxb_ctx ctx, const gvxb_conv_stats_args* a) {
    using namespace gvxb_impl;
    const gvxb_image& s = a->src;
    if (s.format != GVXB_U8) return fail(GVXB_ERR_INVALID, "conv_stats: source must be U8");
    if (!a->sum || !a->sumsq) return fail(GVXB_ERR_INVALID, "conv_stats: sum scratch required");
    if (a->scale < 1) return fail(GVXB_ERR_INVALID, "conv_stats: scale must be >= 1");
    const int frames = s.frames > 0 ? s.frames : 1;
    ConvStatsParams p;
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

    cudaError_t e = cudaMemsetAsync(a->sum, 0, sizeof(int64_t) * frames, ctx->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(a->sumsq, 0, sizeof(int64_t) * frames, ctx->stream);
    if (e == cudaSuccess && a->hist)
        e = cudaMemsetAsync(a->hist, 0, sizeof(gvxb_value) * frames * static_cast<size_t>(p.bins), ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "conv_stats memset");

    void* fn = nullptr;
    int sh = 0;
    switch (a->ksize) {
    case 3: fn = reinterpret_cast<void*>(&conv_stats_kernel<3>), sh = kStTH + 2; break;
    case 5: fn = reinterpret_cast<void*>(&conv_stats_kernel<5>), sh = kStTH + 4; break;
    case 7: fn = reinterpret_cast<void*>(&conv_stats_kernel<7>), sh = kStTH + 6; break;
    default: return fail(GVXB_ERR_UNSUPPORTED, "conv_stats: ksize must be 3, 5 or 7");
    }
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, kStSW, sh)) return rc;
    const size_t dyn = sizeof(unsigned) * (kStThreads / 32) * static_cast<size_t>(p.bins);
    if (dyn > 48 * 1024) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
        if (e != cudaSuccess) return cuda_fail(e, "conv_stats smem attribute");
    }
    dim3 grid((s.width + kStTW - 1) / kStTW, (s.height + kStTH - 1) / kStTH, frames);
    void* args[] = {&map, &p};
    e = cudaLaunchKernel(fn, grid, dim3(kStThreads), args, dyn, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "conv_stats kernel launch");
    if (int rc = check_launch(ctx, "conv_stats kernel")) return rc;
    if (a->mean || a->stddev) {
        const long long n = static_cast<long long>(s.width) * s.height;
        meanstd_finalize_kernel<<<(frames + 63) / 64, 64, 0, ctx->stream>>>(
            p.sum, p.sumsq, n, frames, a->mean, a->stddev);
        if (int rc = check_launch(ctx, "meanstd finalize")) return rc;
    }
    return GVXB_OK;
}
