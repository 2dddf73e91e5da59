// K2 — fused Harris corner graph (U8 -> U8 mask), one pass, sm_100a.
//
// Graph (SURVEY.md §8a "Harris graph definition"): Sobel3x3 -> Multiply
// (gx*gx, gy*gy, gx*gy -> S32) -> Box3x3 (S32) -> user point
// HarrisResponse F32((Sxx*Syy - Sxy^2) - k*(Sxx+Syy)^2) -> user point
// ThresholdF32 sat_U8(resp > T ? 255 : 0).
//
// Exactness argument (the kernel output is bit-identical to run_naive):
//  * Sobel |g| <= 1020, products <= 1020^2, box sums s <= 9*1020^2 < 2^24:
//    every value up to the box sums is an integer held EXACTLY in fp32, so
//    the Sobel / product / box stages run as packed FP32 (FFMA2/FADD2/FMUL2).
//  * The reference rounds each box sum, q = sat_S32(llround(s * (1/9.0)))
//    = round_half_away(s / 9) (ref:src/registry.cpp:703-720), then evaluates
//    the response in int64 + IEEE double (ref:src/expr.cpp:351-371).  With
//    |q - s/9| <= 1/2 and |s_xy| <= (s_xx + s_yy)/2 (Cauchy-Schwarz on the
//    box sums), |81*resp(q) - (s_xx*s_yy - s_xy^2 - k*(s_xx+s_yy)^2)| <=
//    (9 + 18|k|)*tr + 40.5 + 81|k|; adding the fp32 evaluation error
//    (<= 2^-20 * (|p1| + |p2| + |k| tt)) and the float rounding of the final
//    response gives a bound E per pixel.  If |est - 81 T| > E the decision is
//    certain; otherwise (and for every pixel when the F32 response image is
//    observable) the kernel evaluates the reference's exact int64/double
//    expression for that pixel.
//  * Clamp borders of the intermediates: products at out-of-image positions
//    take the clamped position's value (ref:src/execute.cpp:242-245).
//
// Layout: CTA = 4 warps; a warp covers 30 owner lanes x 4 columns (lanes 0
// and 31 are halo lanes whose products reach their neighbours through warp
// shuffles), 64 rows per CTA streamed with 3-row register rings.  Columns
// are kept as even/odd float2 pairs ((c, c+2), (c+1, c+3)) so every
// separable stencil step is a packed, register-aligned FP32 op.
#include "packed.cuh"

#include <cmath>
#include <type_traits>

namespace gvxd {

constexpr int kHarThreads = 128;
constexpr int kHarWarpCols = 120;                         // 30 owner lanes x 4
constexpr int kHarTW = kHarWarpCols * (kHarThreads / 32); // 480 output columns per CTA
constexpr int kHarTH = 64;
constexpr int kHarSW = kHarTW + 32; // smem columns [x0 - 16, x0 + 496): box x start 16-byte aligned
constexpr int kHarSH = kHarTH + 4;  // smem rows    [y0 - 2, y0 + 66)

struct HarrisParams {
    int width;
    int th; // output rows per tile (<= kHarTH), chosen to fill whole waves
    Band band;
    uint8_t* mask;
    int64_t mask_pitch, mask_fstride;
    float* resp;
    int64_t resp_pitch, resp_fstride;
    double k;
    double threshold;
    float kabs;  // |k|
    float kneg;  // -k
    float t81;   // 81 T
    float c_tt;  // bound slope in tt = tr^2
    float c_tr;  // bound slope in tr
    float c0;    // bound constant
};

struct Prod3 {
    Q4 xx, yy, xy; // horizontal box sums of one product row
};
__device__ __forceinline__ Prod3 padd(const Prod3& a, const Prod3& b) {
    return Prod3{qadd(a.xx, b.xx), qadd(a.yy, b.yy), qadd(a.xy, b.xy)};
}

/// The reference's exact expression for one pixel from the exact box sums.
__device__ __forceinline__ float exact_response(float sxx, float syy, float sxy, double k) {
    const int qxx = round_div_away(__float2int_rn(sxx), 9);
    const int qyy = round_div_away(__float2int_rn(syy), 9);
    const int qxy = round_div_away(__float2int_rn(sxy), 9);
    const long long det = static_cast<long long>(qxx) * qyy - static_cast<long long>(qxy) * qxy;
    const long long tr = static_cast<long long>(qxx) + qyy;
    return __double2float_rn(__dsub_rn(__ll2double_rn(det), __dmul_rn(k, __ll2double_rn(tr * tr))));
}

template <bool kResp>
__global__ void __launch_bounds__(kHarThreads) harris_kernel(const __grid_constant__ CUtensorMap map,
                                                             HarrisParams p) {
    __shared__ alignas(128) uint8_t tile[kHarSH * kHarSW];
    __shared__ uint64_t bar;

    const int x0 = blockIdx.x * kHarTW;
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
    stage_tile_u8<kHarSW, kHarSH>(tile, &map, &bar, x0 - 16, y0 - 2, frame, W, p.band, p.th + 4);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = x0 + kHarWarpCols * warp + 4 * (lane - 1); // first column of this lane
    const int off = c - (x0 - 16);                           // its smem column
    const bool owner = lane >= 1 && lane <= 30 && c < W;
    const bool left_edge = c == 0;      // column c-1 clamps to column 0
    const bool right_edge = c + 4 >= W; // column c+4 (and maybe own columns) clamp to W-1
    const int last = W - 1 - c;         // index of column W-1 inside this lane (if 0..3)

    uint8_t* mrow = p.mask + frame * p.mask_fstride + static_cast<int64_t>(y0 - p.band.dst_row0) * p.mask_pitch + c;
    char* rrow = reinterpret_cast<char*>(p.resp) + frame * p.resp_fstride +
                 static_cast<int64_t>(y0 - p.band.dst_row0) * p.resp_pitch;
    const float2 two = f2(2.f, 2.f);

    // kEdge: the warp touches the left / right image border (clamped
    // neighbour columns); interior warps run without those selects
    auto body = [&](auto edge_tag) {
        constexpr bool kEdge = decltype(edge_tag)::value;
        /// Separable Sobel terms of smem row j: D = in(x+1) - in(x-1),
        /// S = in(x-1) + 2 in(x) + in(x+1) for columns c .. c+3.
        /// Source row j as magic floats 2^23 + x in column pairs
        /// P1=(c-1, c+1) P2=(c, c+2) P3=(c+1, c+3) P4=(c+2, c+4): byte
        /// permutes only.  Every use below is a difference of two such
        /// floats, where the 2^23 cancels exactly, so no conversion op.
        auto raw_pairs = [&](int j) {
            const uint8_t* row = tile + j * kHarSW;
            const uint32_t wl = lds32(row, off - 4), wc = lds32(row, off), wr = lds32(row, off + 4);
            Cols6 q;
            q.p1 = f2(magic_byte(wl, 3), magic_byte(wc, 1));
            q.p2 = f2(magic_byte(wc, 0), magic_byte(wc, 2));
            q.p3 = f2(magic_byte(wc, 1), magic_byte(wc, 3));
            q.p4 = f2(magic_byte(wc, 2), magic_byte(wr, 0));
            return q;
        };
        /// Sobel-x row term D = in(x+1) - in(x-1) of source row j.
        auto sobel_d = [&](const Cols6& q) { return Q4{sub2(q.p3, q.p1), sub2(q.p4, q.p2)}; };
        /// Sobel-y of the row between source rows j and j-2: vertical
        /// difference first, then the 1-2-1 smoothing across columns.
        auto sobel_y = [&](const Cols6& q, const Cols6& m) {
            const float2 v1 = sub2(q.p1, m.p1), v2 = sub2(q.p2, m.p2), v3 = sub2(q.p3, m.p3),
                         v4 = sub2(q.p4, m.p4);
            return Q4{fma2(two, v2, add2(v1, v3)), fma2(two, v3, add2(v2, v4))};
        };
        /// Own columns beyond W-1 take column W-1's value (right border clamp).
        auto clamp_right = [&](Q4& q) {
            float v[4] = {q.e.x, q.o.x, q.e.y, q.o.y};
#pragma unroll
            for (int i = 1; i < 4; ++i)
                if (i > last) v[i] = v[i - 1];
            q = Q4{f2(v[0], v[2]), f2(v[1], v[3])};
        };
        /// Horizontal 3-sums; neighbour columns c-1 / c+4 come from adjacent lanes.
        auto hsum = [&](Q4 q) {
            float pm1 = __shfl_up_sync(0xffffffffu, q.o.y, 1);  // left lane's c+3 = my c-1
            float p4 = __shfl_down_sync(0xffffffffu, q.e.x, 1); // right lane's c  = my c+4
            if (kEdge) {
                pm1 = left_edge ? q.e.x : pm1;
                p4 = right_edge ? q.o.y : p4;
            }
            const float2 t = add2(q.e, q.o);
            return Q4{add2(t, f2(pm1, q.o.x)), add2(t, f2(q.e.y, p4))};
        };
        /// Products of one Sobel row and their horizontal box sums.
        auto products = [&](Q4 gx, Q4 gy) {
            Q4 xx = qmul(gx, gx), yy = qmul(gy, gy), xy = qmul(gx, gy);
            if (kEdge && right_edge && last < 3) {
                clamp_right(xx);
                clamp_right(yy);
                clamp_right(xy);
            }
            return Prod3{hsum(xx), hsum(yy), hsum(xy)};
        };
        /// Threshold decision (and optional exact response) for one output row.
        auto emit = [&](int orow, const Prod3& V) {
            const float sxx[4] = {V.xx.e.x, V.xx.o.x, V.xx.e.y, V.xx.o.y};
            const float syy[4] = {V.yy.e.x, V.yy.o.x, V.yy.e.y, V.yy.o.y};
            const float sxy[4] = {V.xy.e.x, V.xy.o.x, V.xy.e.y, V.xy.o.y};
            uint32_t packed = 0;
            float rv[4];
            if constexpr (kResp) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    rv[i] = exact_response(sxx[i], syy[i], sxy[i], p.k);
                    packed |= (static_cast<double>(rv[i]) > p.threshold ? 255u : 0u) << (8 * i);
                }
            } else {
                // certified fp32 estimate of 81 (resp - T); p1 + p2 <= tt / 2
                const float2 kn = f2(p.kneg, p.kneg);
                const float2 ctt = f2(p.c_tt, p.c_tt), c0 = f2(p.c0, p.c0);
                const Q4 tr = qadd(V.xx, V.yy), tt = qmul(tr, tr);
                // det = xx yy - xy^2 with one rounding less (FMA), error within the bound
                // with 81 T folded into the xy^2 term: d = xx yy - (xy^2 + 81 T) - k tt
                const float2 t81 = f2(p.t81, p.t81);
                const float2 qE = fma2(V.xy.e, V.xy.e, t81), qO = fma2(V.xy.o, V.xy.o, t81);
                const Q4 det{fma2(V.xx.e, V.yy.e, f2(-qE.x, -qE.y)), fma2(V.xx.o, V.yy.o, f2(-qO.x, -qO.y))};
                const float2 dE = fma2(kn, tt.e, det.e), dO = fma2(kn, tt.o, det.o);
                // bound linear in tt: the tr term folded in by tr <= (tt / a + a) / 2 (host picks a)
                const float2 eE = fma2(ctt, tt.e, c0), eO = fma2(ctt, tt.o, c0);
                const float d[4] = {dE.x, dO.x, dE.y, dO.y};
                const float e[4] = {eE.x, eO.x, eE.y, eO.y};
                bool unsure = false;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    unsure |= !(fabsf(d[i]) > e[i]);
                    packed |= (d[i] > 0.f ? 255u : 0u) << (8 * i);
                }
                // rare, warp-uniform: the reference's exact expression where the
                // estimate cannot decide
                if (__any_sync(0xffffffffu, unsure)) {
                    packed = 0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        bool on;
                        if (fabsf(d[i]) > e[i]) on = d[i] > 0.f;
                        else on = static_cast<double>(exact_response(sxx[i], syy[i], sxy[i], p.k)) > p.threshold;
                        packed |= (on ? 255u : 0u) << (8 * i);
                    }
                }
                (void)rv;
            }
            if (!owner) return;
            uint8_t* mp = mrow + static_cast<int64_t>(orow) * p.mask_pitch;
            if (!kEdge || c + 3 < W) {
                *reinterpret_cast<uint32_t*>(mp) = packed;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (c + i < W) mp[i] = static_cast<uint8_t>(packed >> (8 * i));
            }
            if constexpr (kResp) {
                float* rp = reinterpret_cast<float*>(rrow + static_cast<int64_t>(orow) * p.resp_pitch) + c;
                if (!kEdge || c + 3 < W) {
                    *reinterpret_cast<float4*>(rp) = make_float4(rv[0], rv[1], rv[2], rv[3]);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (c + i < W) rp[i] = rv[i];
                }
            }
        };

        // Running sums instead of 3-row rings:
        //   gx(r-1) = Q(r-1) + Q(r) with Q(r) = D(r-1) + D(r)
        //   gy(r-1) = T(r-1) + T(r) with T(r) = S(r) - S(r-1)
        //   box(m-1) = P(m-1) + H(m) with P(m) = H(m-1) + H(m)
        // smem row j <-> global y0-2+j; Sobel row j-1 -> product row j-1 ->
        // output row j-2 (global y0-4+j) once j >= 4.
        // State of the running sums, in two alternating copies (A, B) so the
        // 2x-unrolled loop renames instead of moving registers.
        struct State {
            Q4 Dp, Qp;   // D(r-1), Q(r-1)
            Cols6 Raw;   // raw pairs of the source row this copy last consumed
            Prod3 P, Hp; // P(m-1), H(m-1)
        };
        State A, B;
        {
            B.Raw = raw_pairs(0); // the copies alternate, so each holds row j-2 when step j reads it
            A.Raw = raw_pairs(1);
            const Q4 D0 = sobel_d(B.Raw), D1 = sobel_d(A.Raw);
            A.Qp = qadd(D0, D1);
            A.Dp = D1;
        }
        /// Sobel row j-1 from source rows j-2 .. j; writes the successor state into `o`.
        auto sobel_step = [&](int j, const State& i, State& o) {
            const Cols6 q = raw_pairs(j);
            const Q4 D = sobel_d(q);
            const Q4 gy = sobel_y(q, o.Raw); // o.Raw = source row j-2
            o.Raw = q;
            o.Qp = qadd(i.Dp, D);
            o.Dp = D;
            return products(qadd(i.Qp, o.Qp), gy);
        };
        // product rows global y0-1 and y0 (row -1 clamps to row 0 at the top)
        {
            const Prod3 H1 = sobel_step(2, A, B);
            const Prod3 H2 = sobel_step(3, B, A);
            A.P = padd(y0 == 0 ? H2 : H1, H2);
            A.Hp = H2;
        }
        auto full_step = [&](int j, const State& i, State& o) {
            const Prod3 Hn = sobel_step(j, i, o);
            emit(j - 4, padd(i.P, Hn));
            o.P = padd(i.Hp, Hn);
            o.Hp = Hn;
        };
        auto last_step = [&](int j, const State& i, State& o) {
            // product row H clamps to row H-1 at the bottom border
            const Prod3 Hn = sobel_step(j, i, o);
            emit(j - 4, padd(i.P, (y1 == H) ? i.Hp : Hn));
        };
        const int steps = (y1 - y0) + 4;
        int j = 4;
        for (; j + 2 < steps; j += 2) {
            full_step(j, A, B);
            full_step(j + 1, B, A);
        }
        if (j + 1 < steps) {
            full_step(j, A, B);
            last_step(j + 1, B, A);
        } else {
            last_step(j, A, B);
        }
    };
    if (__any_sync(0xffffffffu, left_edge || right_edge)) body(std::true_type{});
    else body(std::false_type{});
}

} // namespace gvxd

using namespace gvxd;

extern "C" int gvxb_harris(gvxb_ctx ctx, const gvxb_harris_args* a) {
    using namespace gvxb_impl;
    const gvxb_image& s = a->src;
    if (s.format != GVXB_U8) return fail(GVXB_ERR_INVALID, "harris: source must be U8");
    if (!a->mask.data) return fail(GVXB_ERR_INVALID, "harris: mask output required");
    const int rows = a->band.row1 - a->band.row0;
    if (rows <= 0 || s.width <= 0) return GVXB_OK;
    HarrisParams p;
    const int frames = s.frames > 0 ? s.frames : 1;
    void* fn = a->response.data ? reinterpret_cast<void*>(&harris_kernel<true>)
                                : reinterpret_cast<void*>(&harris_kernel<false>);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kHarThreads, 0);
    const long long strips = static_cast<long long>(frames) * ((s.width + kHarTW - 1) / kHarTW);
    p.th = balanced_tile_rows(strips, rows, static_cast<long long>(per_sm) * ctx->sm_count, kHarTH, 4);
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, kHarSW, p.th + 4)) return rc;
    p.width = s.width;
    p.band = Band{a->band.row0, a->band.row1, a->band.global_h, a->band.src_row0, a->band.dst_row0};
    p.mask = static_cast<uint8_t*>(a->mask.data);
    p.mask_pitch = a->mask.pitch;
    p.mask_fstride = a->mask.frames > 1 ? a->mask.frame_stride : a->mask.pitch * a->mask.height;
    p.resp = static_cast<float*>(a->response.data);
    p.resp_pitch = a->response.pitch;
    p.resp_fstride = a->response.frames > 1 ? a->response.frame_stride : a->response.pitch * a->response.height;
    p.k = a->k;
    p.threshold = a->threshold;
    const double ak = a->k < 0 ? -a->k : a->k;
    const double at = a->threshold < 0 ? -a->threshold : a->threshold;
    p.kabs = static_cast<float>(ak);
    p.kneg = static_cast<float>(-a->k);
    p.t81 = static_cast<float>(81.0 * a->threshold);
    // rounding perturbation (9 + 18|k|) tr + 40.5 + 81|k| plus the float
    // representation errors of k and 81 T and the final float rounding of
    // the response (|81 T| 2^-22); slack factors keep every term conservative
    // (fl(tr) may be off by 1 above 2^24: +2|k| tr for the tt perturbation)
    const double c_tr = (9.0 + 20.0 * ak) * 1.01 + 1.0;
    // fp32 evaluation error <= 2^-20 (p1 + p2 + |k| tt) <= 2^-20 (1/2 + |k|) tt
    const double c_tt = std::ldexp(0.5 + ak, -20) * 1.01;
    const double c_0 = (40.5 + 81.0 * ak) * 1.1 + 81.0 * at * 5e-7 + 64.0;
    // c_tr tr <= c_tr (tt / a + a) / 2 for any a > 0; the bound is tightest at
    // tr = a, so take a = the smallest tr that can reach the threshold
    // (det <= tt / 4, hence tt >= 81 T / (1/4 - k) on the decision boundary)
    double a_tr = 1.0;
    if (a->threshold > 0 && a->k < 0.24) a_tr = std::sqrt(81.0 * a->threshold / (0.25 - a->k));
    if (!(a_tr >= 1.0) || !std::isfinite(a_tr)) a_tr = 1.0;
    p.c_tr = static_cast<float>(c_tr);
    p.c_tt = static_cast<float>((c_tt + c_tr / (2.0 * a_tr)) * 1.001);
    p.c0 = static_cast<float>((c_0 + c_tr * a_tr / 2.0) * 1.001 + 1.0);
    dim3 grid((s.width + kHarTW - 1) / kHarTW, (rows + p.th - 1) / p.th, frames);
    void* args[] = {&map, &p};
    cudaError_t e = cudaLaunchKernel(fn, grid, dim3(kHarThreads), args, 0, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "harris kernel launch");
    return check_launch(ctx, "harris kernel");
}
