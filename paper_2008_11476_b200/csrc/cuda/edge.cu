// K1 — fused Gaussian3x3 -> Sobel3x3 -> Magnitude (U8 -> S16), one pass.
//
// Reference semantics reproduced bit-exactly:
//   gaussian3x3  sat_U8(llround(s * (1/16))) == floor((s + 8) / 16), s <= 4080
//                (ref:src/registry.cpp:722-746)
//   sobel_x/y    sat_S16(sum(mask * win)), |v| <= 1020 (ref:src/registry.cpp:748-784)
//   magnitude    sat_S16(llround(sqrt((double)(gx^2 + gy^2))))
//                (ref:src/registry.cpp:555-575): fp32 estimate + exact
//                integer correction, n = gx^2 + gy^2 < 2^22
//   Clamp of the *intermediate*: the Gaussian at an out-of-image position is
//   the Gaussian of the clamped position (run_naive materialises it and the
//   Sobel window clamps into it, ref:src/execute.cpp:242-245).
// Every intermediate is an integer < 2^24, so the pipeline runs on packed
// FP32 (FFMA2/FADD2/FMUL2) with exact arithmetic; see packed.cuh.
//
// Layout: CTA = 4 warps, 30 owner lanes x 4 columns per warp (lanes 0 / 31
// are halo lanes whose Gaussian columns reach their neighbours by warp
// shuffles), 64 output rows per CTA streamed with running sums:
//   Gaussian  v(r-1) = R(r-1) + R(r),  R(r) = Hg(r-1) + Hg(r)
//   Sobel     gx(r-1) = Q(r-1) + Q(r), Q(r) = D(r-1) + D(r)
//             gy(r-1) = T(r-1) + T(r), T(r) = S(r) - S(r-1)
// so every input byte is read from HBM once (+ a 4-row halo) and every
// output written once: 1 B in + 2 B out per output pixel.
#include "packed.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace gvxd {

constexpr int kEdgeThreads = 128;
constexpr int kEdgeWarpCols = 120;
constexpr int kEdgeTW = kEdgeWarpCols * (kEdgeThreads / 32); // 480
#ifndef GVX_EDGE_TH_MAX
#define GVX_EDGE_TH_MAX 40
#endif
constexpr int kEdgeTH = GVX_EDGE_TH_MAX; // measured best of 24..64 (occupancy vs halo rows)
constexpr int kEdgeSW = kEdgeTW + 32; // smem columns [x0 - 16, x0 + 496)
constexpr int kEdgeSH = kEdgeTH + 4;  // smem rows    [y0 - 2, y0 + 66)

struct OutPlane {
    int16_t* data;
    int64_t pitch;        // bytes
    int64_t frame_stride; // bytes
};

struct EdgeParams {
    int width;
    int th; // output rows per tile (<= kEdgeTH), chosen to fill whole waves
    Band band;
    OutPlane gx, gy, mag;
};

/// Integer-valued floats |v| < 2^22 to int16 pairs packed in a u32.
__device__ __forceinline__ uint32_t pack_s16(float lo, float hi) {
    const float m = 12582912.f; // 1.5 * 2^23: low mantissa bits = two's complement value
    return __byte_perm(__float_as_uint(lo + m), __float_as_uint(hi + m), 0x5410);
}

/// Four S16 columns at p (columns c .. c+3); `full` = all inside the image.
__device__ __forceinline__ void store4p(int16_t* p, bool full, int nvalid, Q4 v) {
    if (full) {
        *reinterpret_cast<uint2*>(p) = make_uint2(pack_s16(v.e.x, v.o.x), pack_s16(v.e.y, v.o.y));
    } else {
        const float vv[4] = {v.e.x, v.o.x, v.e.y, v.o.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (i < nvalid) p[i] = static_cast<int16_t>(__float2int_rn(vv[i]));
    }
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

/// round(sqrt(n)) half away from zero for integer-valued 0 <= n < 2^22:
/// k0 = floor(s + 0.49) in {k*-1, k*} for the approximate s, then
/// k* = k0 + (n > k0^2 + k0) (k* is the largest k with k^2 - k < n).
__device__ __forceinline__ Q4 round_sqrt4(Q4 n) {
    const float2 M = f2(12582912.f, 12582912.f), nM = f2(-12582912.f, -12582912.f), d = f2(-0.01f, -0.01f);
    const Q4 s{f2(sqrt_approx(n.e.x), sqrt_approx(n.e.y)), f2(sqrt_approx(n.o.x), sqrt_approx(n.o.y))};
    Q4 k{add2(add2(add2(s.e, d), M), nM), add2(add2(add2(s.o, d), M), nM)};
    const Q4 kk{fma2(k.e, k.e, k.e), fma2(k.o, k.o, k.o)};
    k.e.x += n.e.x > kk.e.x ? 1.f : 0.f;
    k.e.y += n.e.y > kk.e.y ? 1.f : 0.f;
    k.o.x += n.o.x > kk.o.x ? 1.f : 0.f;
    k.o.y += n.o.y > kk.o.y ? 1.f : 0.f;
    return k;
}

template <bool kGauss, bool kGx, bool kGy, bool kMag>
__global__ void __launch_bounds__(kEdgeThreads) edge_kernel(const __grid_constant__ CUtensorMap map, EdgeParams p) {
    __shared__ alignas(128) uint8_t tile[kEdgeSH * kEdgeSW];
    __shared__ uint64_t bar;

    const int x0 = blockIdx.x * kEdgeTW;
    const int y0 = p.band.row0 + blockIdx.y * p.th;
    const int y1 = min(y0 + p.th, p.band.row1);
    const int frame = blockIdx.z;
    const int H = p.band.global_h;
    const int W = p.width;

    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    stage_tile_u8<kEdgeSW, kEdgeSH>(tile, &map, &bar, x0 - 16, y0 - 2, frame, W, p.band, p.th + 4);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = x0 + kEdgeWarpCols * warp + 4 * (lane - 1);
    const int off = c - (x0 - 16);
    const bool owner = lane >= 1 && lane <= 30 && c < W;
    const bool left_edge = c == 0;
    const bool right_edge = c + 4 >= W;
    const int last = W - 1 - c;
    const int orow0 = y0 - p.band.dst_row0;

    // kEdge: the warp touches the left / right image border (clamped
    // neighbour columns, partial stores); interior warps skip that code
    auto body = [&](auto edge_tag) {
        constexpr bool kEdge = decltype(edge_tag)::value;
        // output row pointers advance one row per emit (rows are emitted in order)
        auto row_ptr = [&](const OutPlane& o) {
            return reinterpret_cast<int16_t*>(reinterpret_cast<char*>(o.data) + frame * o.frame_stride +
                                              static_cast<int64_t>(orow0) * o.pitch) + c;
        };
        int16_t* pgx = kGx ? row_ptr(p.gx) : nullptr;
        int16_t* pgy = kGy ? row_ptr(p.gy) : nullptr;
        int16_t* pmag = kMag ? row_ptr(p.mag) : nullptr;
        const bool full = c + 3 < W;
        const int nvalid = W - c;
        auto emit = [&](Q4 gx, Q4 gy) {
            if (owner) {
                const bool f = !kEdge || full;
                if (kGx) store4p(pgx, f, nvalid, gx);
                if (kGy) store4p(pgy, f, nvalid, gy);
                if (kMag)
                    store4p(pmag, f, nvalid,
                            round_sqrt4(Q4{fma2(gx.e, gx.e, mul2(gy.e, gy.e)), fma2(gx.o, gx.o, mul2(gy.o, gy.o))}));
            }
            if (kGx) pgx = reinterpret_cast<int16_t*>(reinterpret_cast<char*>(pgx) + p.gx.pitch);
            if (kGy) pgy = reinterpret_cast<int16_t*>(reinterpret_cast<char*>(pgy) + p.gy.pitch);
            if (kMag) pmag = reinterpret_cast<int16_t*>(reinterpret_cast<char*>(pmag) + p.mag.pitch);
        };

        struct State {
            Q4 Dp, Qp, Sp, Tp; // Sobel running sums over the (Gaussian) rows
            Q4 Hp, Rp;         // Gaussian running sums over source rows
        };
        State A, B;

        if constexpr (kGauss) {
            const float2 sc = f2(0.0625f, 0.0625f), M = f2(12582912.f, 12582912.f);
            const float2 nM = f2(-12582912.f, -12582912.f);
            /// Gaussian row (exact) from the biased sum v' = v + 8 (the +8 rides
            /// in the source conversion, see load_cols6_biased):
            /// floor(v' / 16) = fma_rd(v', 1/16, 1.5 * 2^23) - 1.5 * 2^23.
            auto gauss_round = [&](Q4 v) {
                return Q4{add2(__ffma2_rd(v.e, sc, M), nM), add2(__ffma2_rd(v.o, sc, M), nM)};
            };
            /// Sobel row terms of a Gaussian row held in registers (neighbour
            /// columns through shuffles, clamped at the image border).
            auto gauss_sobel_terms = [&](Q4 g, Q4& D, Q4& S) {
                if (kEdge && right_edge && last < 3) {
                    float v[4] = {g.e.x, g.o.x, g.e.y, g.o.y};
#pragma unroll
                    for (int i = 1; i < 4; ++i)
                        if (i > last) v[i] = v[i - 1];
                    g = Q4{f2(v[0], v[2]), f2(v[1], v[3])};
                }
                float gl = __shfl_up_sync(0xffffffffu, g.o.y, 1);
                float gr = __shfl_down_sync(0xffffffffu, g.e.x, 1);
                if (kEdge) {
                    gl = left_edge ? g.e.x : gl;
                    gr = right_edge ? g.o.y : gr;
                }
                diff_smooth(neighbourhood(g, gl, gr), D, S);
            };
            /// Source row j: Gaussian horizontal sums; returns the Gaussian row
            /// centred one row up (smem row j-1).
            auto src_step = [&](int j, const State& i, State& o) {
                Q4 Dn, Hg;
                diff_smooth(load_cols6_biased(tile + j * kEdgeSW, off), Dn, Hg); // Hg + 2 (Dn unused)
                o.Rp = qadd(i.Hp, Hg);
                o.Hp = Hg;
                return gauss_round(qadd(i.Rp, o.Rp));
            };
            {
                Q4 Dn, S0, S1;
                diff_smooth(load_cols6_biased(tile, off), Dn, S0);
                diff_smooth(load_cols6_biased(tile + kEdgeSW, off), Dn, S1);
                A.Hp = S1;
                A.Rp = qadd(S0, S1);
            }
            Q4 D1, G1, D2, G2;
            gauss_sobel_terms(src_step(2, A, B), D1, G1); // Gaussian row y0-1
            gauss_sobel_terms(src_step(3, B, A), D2, G2); // Gaussian row y0
            if (y0 == 0) {                                // Gaussian row -1 clamps to row 0
                D1 = D2;
                G1 = G2;
            }
            A.Qp = qadd(D1, D2);
            A.Tp = qsub(G2, G1);
            A.Dp = D2;
            A.Sp = G2;
            auto full_step = [&](int j, const State& i, State& o, bool bottom) {
                Q4 D, S;
                gauss_sobel_terms(src_step(j, i, o), D, S);
                if (bottom) { // Gaussian row H clamps to row H-1
                    D = i.Dp;
                    S = i.Sp;
                }
                o.Qp = qadd(i.Dp, D);
                o.Tp = qsub(S, i.Sp);
                o.Dp = D;
                o.Sp = S;
                emit(qadd(i.Qp, o.Qp), qadd(i.Tp, o.Tp));
            };
            const int steps = (y1 - y0) + 4;
            int j = 4;
            for (; j + 2 < steps; j += 2) {
                full_step(j, A, B, false);
                full_step(j + 1, B, A, false);
            }
            const bool bot = y1 == H;
            if (j + 1 < steps) {
                full_step(j, A, B, false);
                full_step(j + 1, B, A, bot);
            } else {
                full_step(j, A, B, bot);
            }
        } else {
            // Sobel straight on the source (Clamp is already in shared memory)
            {
                Q4 D0, S0, D1, S1;
                diff_smooth(load_cols6(tile + 1 * kEdgeSW, off), D0, S0); // global y0-1
                diff_smooth(load_cols6(tile + 2 * kEdgeSW, off), D1, S1); // global y0
                A.Qp = qadd(D0, D1);
                A.Tp = qsub(S1, S0);
                A.Dp = D1;
                A.Sp = S1;
            }
            auto step = [&](int j, const State& i, State& o) {
                Q4 D, S;
                diff_smooth(load_cols6(tile + j * kEdgeSW, off), D, S);
                o.Qp = qadd(i.Dp, D);
                o.Tp = qsub(S, i.Sp);
                o.Dp = D;
                o.Sp = S;
                emit(qadd(i.Qp, o.Qp), qadd(i.Tp, o.Tp));
            };
            const int steps = (y1 - y0) + 3;
            int j = 3;
            for (; j + 1 < steps; j += 2) {
                step(j, A, B);
                step(j + 1, B, A);
            }
            if (j < steps) step(j, A, B);
        }
    };
    if (__any_sync(0xffffffffu, left_edge || right_edge)) body(std::true_type{});
    else body(std::false_type{});
}

} // namespace gvxd

using namespace gvxd;

namespace {

OutPlane plane(const gvxb_image& img) {
    OutPlane o;
    o.data = static_cast<int16_t*>(img.data);
    o.pitch = img.pitch;
    o.frame_stride = img.frames > 1 ? img.frame_stride : img.pitch * img.height;
    return o;
}

template <bool G>
void* pick_edge(bool ox, bool oy, bool om) {
    const int code = (ox ? 4 : 0) | (oy ? 2 : 0) | (om ? 1 : 0);
    switch (code) {
    case 1: return reinterpret_cast<void*>(&edge_kernel<G, false, false, true>);
    case 2: return reinterpret_cast<void*>(&edge_kernel<G, false, true, false>);
    case 3: return reinterpret_cast<void*>(&edge_kernel<G, false, true, true>);
    case 4: return reinterpret_cast<void*>(&edge_kernel<G, true, false, false>);
    case 5: return reinterpret_cast<void*>(&edge_kernel<G, true, false, true>);
    case 6: return reinterpret_cast<void*>(&edge_kernel<G, true, true, false>);
    case 7: return reinterpret_cast<void*>(&edge_kernel<G, true, true, true>);
    default: return nullptr;
    }
}

} // namespace

namespace gvxb_impl {
int edge8_launch(gvxb_ctx ctx, const gvxb_edge_args* a); // edge8.cu
}

extern "C" int gvxb_edge(gvxb_ctx ctx, const gvxb_edge_args* a) {
    using namespace gvxb_impl;
    const gvxb_image& s = a->src;
    if (s.format != GVXB_U8) return fail(GVXB_ERR_INVALID, "edge: source must be U8");
    const bool ox = a->gx.data, oy = a->gy.data, om = a->mag.data;
    void* fn = a->with_gauss ? pick_edge<true>(ox, oy, om) : pick_edge<false>(ox, oy, om);
    if (!fn) return GVXB_OK; // nothing requested
    const int rows = a->band.row1 - a->band.row0;
    if (rows <= 0 || s.width <= 0) return GVXB_OK;
    // Gaussian graphs run the one-warp / 8-column kernel (edge8.cu);
    // GVX_EDGE_V2=1 selects this file's 4-warp tiled kernel (A/B tests)
    static const bool v2 = std::getenv("GVX_EDGE_V2") != nullptr;
    if (a->with_gauss && !v2) return edge8_launch(ctx, a);
    const int frames = s.frames > 0 ? s.frames : 1;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kEdgeThreads, 0);
    const long long strips = static_cast<long long>(frames) * ((s.width + kEdgeTW - 1) / kEdgeTW);
    EdgeParams p;
    p.th = balanced_tile_rows(strips, rows, static_cast<long long>(per_sm) * ctx->sm_count, kEdgeTH, 4);
    if (const char* e = std::getenv("GVX_EDGE_TH")) p.th = std::max(8, std::min(kEdgeTH, std::atoi(e))); // tuning experiments
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, kEdgeSW, p.th + 4)) return rc;
    p.width = s.width;
    p.band = Band{a->band.row0, a->band.row1, a->band.global_h, a->band.src_row0, a->band.dst_row0};
    p.gx = plane(a->gx);
    p.gy = plane(a->gy);
    p.mag = plane(a->mag);
    dim3 grid((s.width + kEdgeTW - 1) / kEdgeTW, (rows + p.th - 1) / p.th, frames);
    void* args[] = {&map, &p};
    untracked_op(ctx);
    cudaError_t e = cudaLaunchKernel(fn, grid, dim3(kEdgeThreads), args, 0, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "edge kernel launch");
    return check_launch(ctx, "edge kernel");
}
