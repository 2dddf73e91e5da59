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
// Layout (v4): one warp per CTA owns a strip of 248 output columns and a
// band of rows.  Lane L holds 8 columns c = x - 4 + 8L .. c + 7 as four
// float2 pairs (A_i, B_i) = (column c+i, column c+4+i): every stencil step
// is then a plain packed op on register pairs with no lane-internal
// shuffling of halves, and only the strip's outer half-lanes (lane 0's A
// half, lane 31's B half) are halo.  Source rows stream through a 16-row
// shared-memory ring filled by 8-row TMA chunks, so a band pays its 4 halo
// rows once however tall it is.
#include "packed.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

namespace gvxd {

constexpr int kHarThreads = 32;  // one warp per CTA
constexpr int kHarCols = 248;    // output columns per strip (32 lanes x 8 - 8 halo)
constexpr int kHarSW = 288;      // ring row bytes: image columns [x_org, x_org + 288)
#ifndef GVX_HARRIS_CHUNK
#define GVX_HARRIS_CHUNK 16 // measured: 16 > 8 (+2.5%) > 4
#endif
constexpr int kHarChunk = GVX_HARRIS_CHUNK; // rows per TMA chunk
constexpr int kHarRing = 2 * kHarChunk;
constexpr int kHarTHMax = 128; // measured with overlapped launches (4K x32): 64 -> 128 rows +2.5%, 192 / 256 less

struct HarrisParams {
    int width;
    int pdl_wait; // the previous grid on the stream may have written what this one touches
    int th; // output rows per band (<= kHarTHMax), chosen to fill whole waves
    Band band;
    uint8_t* mask;
    int64_t mask_pitch, mask_fstride;
    float* resp;
    int64_t resp_pitch, resp_fstride;
    double k;
    double threshold;
    float kpos;  // k
    float t81;   // 81 T
    float c_tt;  // bound slope in tt = tr^2
    float c0;    // bound constant
};

/// Four column pairs (A_i, B_i) = (c+i, c+4+i).
struct Q8 {
    float2 v[4];
};
/// Source pairs for i = -1 .. 4 at v[i + 1] (magic floats 2^15 + x).
struct Raw8 {
    float2 v[6];
};
struct Prod3 {
    Q8 xx, yy, xy;
};
__device__ __forceinline__ Q8 q8add(const Q8& a, const Q8& b) {
    return Q8{{add2(a.v[0], b.v[0]), add2(a.v[1], b.v[1]), add2(a.v[2], b.v[2]), add2(a.v[3], b.v[3])}};
}
__device__ __forceinline__ Q8 q8mul(const Q8& a, const Q8& b) {
    return Q8{{mul2(a.v[0], b.v[0]), mul2(a.v[1], b.v[1]), mul2(a.v[2], b.v[2]), mul2(a.v[3], b.v[3])}};
}
__device__ __forceinline__ Prod3 padd(const Prod3& a, const Prod3& b) {
    return Prod3{q8add(a.xx, b.xx), q8add(a.yy, b.yy), q8add(a.xy, b.xy)};
}
__device__ __forceinline__ uint2 lds64(const uint8_t* p) { return *reinterpret_cast<const uint2*>(p); }

/// 2^15 + byte k of w (the float bit pattern 0x4700bb00; ulp 2^-8): sums of
/// four of them stay below 2^17 + 2^10, where integers are still exact.
__device__ __forceinline__ float magic15_byte(uint32_t w, int k) {
    return __uint_as_float(__byte_perm(w, 0x47000000u, 0x7404u | (static_cast<unsigned>(k) << 4)));
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

/// Bytes 0, 1 = 0xFF where a / b is negative (sign bit set), else 0x00:
/// prmt's sign-replicate selector mode (the __byte_perm intrinsic masks it).
__device__ __forceinline__ uint32_t sign_bytes(float a, float b) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, 0xFBFB;" : "=r"(r) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
    return r;
}

#ifndef GVX_HARRIS_UNROLL
#define GVX_HARRIS_UNROLL 2 // rows per loop iteration of interior strips (measured: 4 rows (two pair steps) -9%)
#endif
#ifndef GVX_HARRIS4_MINB
#define GVX_HARRIS4_MINB 16 // 4-column kernel: 4 warps per scheduler at <= 128 registers
#endif
#ifndef GVX_HARRIS4_UNROLL
#define GVX_HARRIS4_UNROLL 4 // interior strips: two pair steps per iteration (measured +7% over 2 rows)
#endif
template <bool kResp>
#ifndef GVX_HARRIS_MINB
#define GVX_HARRIS_MINB 12 // resident one-warp CTAs per SM: 3 per scheduler at <= 168 registers
#endif
__global__ void __launch_bounds__(kHarThreads, GVX_HARRIS_MINB) harris_kernel(const __grid_constant__ CUtensorMap map,
                                                                 HarrisParams p) {
    __shared__ alignas(128) uint8_t ring[kHarRing * kHarSW];
    __shared__ uint64_t bar[2];

    const int lane = threadIdx.x;
    // first output column of the strip (a multiple of 8: keeps the lanes'
    // 64-bit ring loads aligned); the last strip is pulled left to end at
    // roundup8(W) so that it has no idle lanes (overlapping columns are
    // computed twice, with identical results)
    const int x = max(0, min(static_cast<int>(blockIdx.x) * kHarCols, ((p.width + 7) & ~7) - kHarCols));
    const int x_org = ((x - 5) >> 4) << 4;    // ring column 0 (16-byte aligned TMA origin)
    const int y0 = p.band.row0 + blockIdx.y * p.th;
    const int y1 = min(y0 + p.th, p.band.row1);
    const int frame = blockIdx.z;
    const int H = p.band.global_h;
    const int W = p.width;
    const int steps = (y1 - y0) + 4; // virtual rows j <-> global row y0 - 2 + j
    const int nchunks = (steps + kHarChunk - 1) / kHarChunk;

    pdl_prologue(p.pdl_wait);
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    __syncwarp();

    auto issue = [&](int k) { // lane 0: chunk k -> ring half k & 1
        uint64_t* b = &bar[k & 1];
        mbar_expect_tx(b, kHarChunk * kHarSW);
        tma_load_3d(ring + (k & 1) * kHarChunk * kHarSW, &map, b, x_org / 4,
                    y0 - 2 + kHarChunk * k - p.band.src_row0, frame);
    };
    // Clamp borders of the source: columns outside [0, W) replicate the edge
    // column, rows outside [0, H) the edge row (ref:src/execute.cpp:242-245).
    const bool col_patch = x_org < 0 || x_org + kHarSW > W;
    bool dirty = false; // the ring half about to be refilled holds generic-proxy writes
    auto patch = [&](int k) {
        uint8_t* base = ring + (k & 1) * kHarChunk * kHarSW;
        const int g0 = y0 - 2 + kHarChunk * k;
        const bool rows = g0 < 0 || g0 + kHarChunk > H;
        if (col_patch) {
            // smem columns [0, first) take column first (image column 0),
            // (lastc, kHarSW) take column lastc (image column W-1)
            const int first = clampi(-x_org, 0, kHarSW - 1), lastc = clampi(W - 1 - x_org, 0, kHarSW - 1);
            for (int r = 0; r < kHarChunk; ++r) {
                uint8_t* row = base + r * kHarSW;
                if (lane < first) row[lane] = row[first];
                for (int j = lastc + 1 + lane; j < kHarSW; j += 32) row[j] = row[lastc];
            }
            __syncwarp();
        }
        if (rows) {
            for (int r = 0; r < kHarChunk; ++r) {
                const int gy = g0 + r;
                if ((gy >= 0 && gy < H) || kHarChunk * k + r >= steps) continue;
                const int v = clampi(gy, 0, H - 1) - (y0 - 2); // virtual row of the clamped source row
                const uint32_t* from = reinterpret_cast<const uint32_t*>(ring + (v % kHarRing) * kHarSW);
                uint32_t* to = reinterpret_cast<uint32_t*>(base + r * kHarSW);
                for (int j = lane; j < kHarSW / 4; j += 32) to[j] = from[j];
            }
            __syncwarp();
        }
        return col_patch || rows;
    };
    /// Waits for chunk k, patches its borders, then starts chunk k + 1 into
    /// the other half (whose rows the warp has finished reading).
    auto next_chunk = [&](int k) {
        mbar_wait(&bar[k & 1], (k >> 1) & 1);
        const bool patched = patch(k);
        if (lane == 0 && k + 1 < nchunks) {
            if (dirty) fence_proxy_async_smem();
            issue(k + 1);
        }
        dirty = patched;
    };

    const int c = x - 4 + 8 * lane; // first column of this lane
    const int off = c - x_org;      // its ring column (4 <= off, off % 8 == 4)
    const int last = W - 1 - c;     // index of column W-1 among c .. c+7 (when 0..7)
    const bool store_a = lane > 0 && c < W;
    const bool store_b = lane < 31 && c + 4 < W;

    uint8_t* mrow = p.mask + frame * p.mask_fstride + static_cast<int64_t>(y0 - p.band.dst_row0) * p.mask_pitch + c;
    char* rrow = reinterpret_cast<char*>(p.resp) + frame * p.resp_fstride +
                 static_cast<int64_t>(y0 - p.band.dst_row0) * p.resp_pitch;
    const float2 two = f2(2.f, 2.f);

    if (lane == 0) issue(0);
    next_chunk(0);

    // kEdge: the strip touches the left / right image border (clamped
    // product columns); interior strips run without those selects
    auto body = [&](auto edge_tag) {
        constexpr bool kEdge = decltype(edge_tag)::value;
        /// Source row j as magic floats 2^15 + x (byte permutes only): pairs
        /// for i = -1 .. 4.  Every use ends in a difference of two rows or
        /// columns, where the 2^15 terms cancel exactly.
        auto raw_pairs = [&](int j) {
            const uint8_t* row = ring + (j % kHarRing) * kHarSW + off;
            const uint2 lo = lds64(row - 4), hi = lds64(row + 4); // columns c-4 .. c+3, c+4 .. c+11
            Raw8 r;
            r.v[0] = f2(magic15_byte(lo.x, 3), magic15_byte(lo.y, 3));
            r.v[1] = f2(magic15_byte(lo.y, 0), magic15_byte(hi.x, 0));
            r.v[2] = f2(magic15_byte(lo.y, 1), magic15_byte(hi.x, 1));
            r.v[3] = f2(magic15_byte(lo.y, 2), magic15_byte(hi.x, 2));
            r.v[4] = f2(magic15_byte(lo.y, 3), magic15_byte(hi.x, 3));
            r.v[5] = f2(magic15_byte(hi.x, 0), magic15_byte(hi.y, 0));
            return r;
        };
        /// Sobel-x row term D = in(x+1) - in(x-1).
        auto sobel_d = [&](const Raw8& q) {
            return Q8{{sub2(q.v[2], q.v[0]), sub2(q.v[3], q.v[1]), sub2(q.v[4], q.v[2]), sub2(q.v[5], q.v[3])}};
        };
        /// Horizontal 1-2-1 smoothing S of a source row (values 2^17 + s,
        /// exact); Sobel-y of row j-1 is S(j) - S(j-2).
        auto smooth = [&](const Raw8& q) {
            Q8 g;
#pragma unroll
            for (int i = 0; i < 4; ++i) g.v[i] = fma2(two, q.v[i + 1], add2(q.v[i], q.v[i + 2]));
            return g;
        };
        /// Columns beyond W-1 take column W-1's value; at the left border the
        /// product at column -1 (lane 0's A3) takes column 0's (B0).
        auto clamp_cols = [&](Q8& q) {
            if (!kEdge) return;
            if (last < 7) { // divergent: only the lane holding column W-1 (and idle lanes)
                float v[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    v[i] = q.v[i].x;
                    v[i + 4] = q.v[i].y;
                }
#pragma unroll
                for (int i = 1; i < 8; ++i)
                    if (i > last) v[i] = v[i - 1];
#pragma unroll
                for (int i = 0; i < 4; ++i) q.v[i] = f2(v[i], v[i + 4]);
            }
            if (x == 0 && lane == 0) q.v[3].x = q.v[0].y;
        };
        /// Horizontal 3-sums; columns c-1 / c+8 come from the adjacent lanes.
        auto hsum = [&](const Q8& q) {
            const float L = __shfl_up_sync(0xffffffffu, q.v[3].y, 1); // left lane's B3 = my c-1
            float R = __shfl_down_sync(0xffffffffu, q.v[0].x, 1);     // right lane's A0 = my c+8
            if (kEdge) R = last <= 7 ? q.v[3].y : R;
            const float2 sa = add2(q.v[0], q.v[1]), sb = add2(q.v[2], q.v[3]);
            // the two boundary outputs as scalar adds: assembling the pairs
            // (L, A3) and (B0, R) cost a register move each (measured +2.8%)
            return Q8{{f2(L + sa.x, q.v[3].x + sa.y), add2(sa, q.v[2]), add2(q.v[1], sb), f2(sb.x + q.v[0].y, sb.y + R)}};
        };
        /// Products of one Sobel row and their horizontal box sums.
        auto products = [&](const Q8& gx, const Q8& gy) {
            Q8 xx = q8mul(gx, gx), yy = q8mul(gy, gy), xy = q8mul(gx, gy);
            clamp_cols(xx);
            clamp_cols(yy);
            clamp_cols(xy);
            return Prod3{hsum(xx), hsum(yy), hsum(xy)};
        };
        /// Threshold decision (and optional exact response) for one output row.
        auto emit = [&](const Prod3& V) { // output rows in order, from y0
            uint32_t ma = 0, mb = 0;
            float rv[8];
            if constexpr (kResp) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    rv[i] = exact_response(V.xx.v[i].x, V.yy.v[i].x, V.xy.v[i].x, p.k);
                    rv[i + 4] = exact_response(V.xx.v[i].y, V.yy.v[i].y, V.xy.v[i].y, p.k);
                    ma |= (static_cast<double>(rv[i]) > p.threshold ? 255u : 0u) << (8 * i);
                    mb |= (static_cast<double>(rv[i + 4]) > p.threshold ? 255u : 0u) << (8 * i);
                }
            } else {
                // certified fp32 estimate of -81 (resp - T):
                //   nd = k tt - xx yy + (xy^2 + 81 T), bound e = c_tt tt + c0
                const float2 kk = f2(p.kpos, p.kpos), t81 = f2(p.t81, p.t81);
                const float2 ctt = f2(p.c_tt, p.c_tt), c0 = f2(p.c0, p.c0);
                float2 nd[4], e[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 tr = add2(V.xx.v[i], V.yy.v[i]);
                    const float2 tt = mul2(tr, tr);
                    const float2 w = fma2(V.xy.v[i], V.xy.v[i], t81);
                    const float2 ndet = fma2(f2(-V.xx.v[i].x, -V.xx.v[i].y), V.yy.v[i], w);
                    nd[i] = fma2(kk, tt, ndet);
                    e[i] = fma2(ctt, tt, c0);
                }
                bool unsure = false;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    unsure |= !(fabsf(nd[i].x) > e[i].x);
                    unsure |= !(fabsf(nd[i].y) > e[i].y);
                }
                // mask byte = sign of nd replicated (nd < 0 <=> resp > T)
                const uint32_t a01 = sign_bytes(nd[0].x, nd[1].x), a23 = sign_bytes(nd[2].x, nd[3].x);
                const uint32_t b01 = sign_bytes(nd[0].y, nd[1].y), b23 = sign_bytes(nd[2].y, nd[3].y);
                ma = __byte_perm(a01, a23, 0x5410);
                mb = __byte_perm(b01, b23, 0x5410);
                // rare, warp-uniform: the reference's exact expression where the
                // estimate cannot decide
                if (__any_sync(0xffffffffu, unsure)) {
                    // one compact loop over this lane's undecided pixels (values
                    // spilled to a local array: the path is rare and kept small)
                    unsigned ub = 0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        ub |= (fabsf(nd[i].x) > e[i].x ? 0u : 1u) << i;
                        ub |= (fabsf(nd[i].y) > e[i].y ? 0u : 1u) << (i + 4);
                    }
                    if (ub) {
                        float buf[24];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            buf[i] = V.xx.v[i].x, buf[i + 4] = V.xx.v[i].y;
                            buf[8 + i] = V.yy.v[i].x, buf[12 + i] = V.yy.v[i].y;
                            buf[16 + i] = V.xy.v[i].x, buf[20 + i] = V.xy.v[i].y;
                        }
#pragma unroll 1
                        while (ub) {
                            const int i = __ffs(ub) - 1;
                            ub &= ub - 1;
                            const bool on =
                                static_cast<double>(exact_response(buf[i], buf[8 + i], buf[16 + i], p.k)) > p.threshold;
                            const int sh = 8 * (i & 3);
                            const uint32_t bit = (on ? 255u : 0u) << sh, keep = ~(255u << sh);
                            if (i < 4) ma = (ma & keep) | bit;
                            else mb = (mb & keep) | bit;
                        }
                    }
                }
                (void)rv;
            }
            uint8_t* mp = mrow;
            mrow += p.mask_pitch;
            if (!kEdge || c + 7 < W) {
                if (store_a) *reinterpret_cast<uint32_t*>(mp) = ma;
                if (store_b) *reinterpret_cast<uint32_t*>(mp + 4) = mb;
            } else { // the lane holding column W-1 (and lanes past it, which store nothing)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (store_a && c + i < W) mp[i] = static_cast<uint8_t>(ma >> (8 * i));
                    if (store_b && c + 4 + i < W) mp[4 + i] = static_cast<uint8_t>(mb >> (8 * i));
                }
            }
            if constexpr (kResp) {
                float* rp = reinterpret_cast<float*>(rrow) + c;
                rrow += p.resp_pitch;
                if (!kEdge || c + 7 < W) {
                    if (store_a) *reinterpret_cast<float4*>(rp) = make_float4(rv[0], rv[1], rv[2], rv[3]);
                    if (store_b) *reinterpret_cast<float4*>(rp + 4) = make_float4(rv[4], rv[5], rv[6], rv[7]);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if (store_a && c + i < W) rp[i] = rv[i];
                        if (store_b && c + 4 + i < W) rp[4 + i] = rv[4 + i];
                    }
                }
            }
        };

        // Running sums (as v3):
        //   gx(r-1) = Q(r-1) + Q(r) with Q(r) = D(r-1) + D(r)
        //   gy(r-1) = S(r) - S(r-2), taken as vertical differences first
        //   box(m-1) = P(m-1) + H(m) with P(m) = H(m-1) + H(m)
        // virtual row j -> Sobel row j-1 -> product row j-1 -> output row
        // j-4 once j >= 4.  Two alternating state copies (A, B) so the
        // 2x-unrolled loop renames instead of moving registers.
        struct State {
            Q8 Dp, Qp;   // D(r-1), Q(r-1)
            Q8 S;        // smoothing S of the source row this copy last consumed
            Prod3 P, Hp; // P(m-1), H(m-1)
        };
        State A, B;
        {
            const Raw8 r0 = raw_pairs(0), r1 = raw_pairs(1);
            B.S = smooth(r0); // the copies alternate, so each holds row j-2 when step j reads it
            A.S = smooth(r1);
            const Q8 D0 = sobel_d(r0), D1 = sobel_d(r1);
            A.Qp = q8add(D0, D1);
            A.Dp = D1;
        }
        /// Sobel row j-1 from source rows j-2 .. j; writes the successor state into `o`.
        auto sobel_step = [&](int j, const State& i, State& o) {
            const Raw8 q = raw_pairs(j);
            const Q8 D = sobel_d(q);
            const Q8 S = smooth(q);
            Q8 gy;
#pragma unroll
            for (int t = 0; t < 4; ++t) gy.v[t] = sub2(S.v[t], o.S.v[t]); // o.S = S of source row j-2
            o.S = S;
            o.Qp = q8add(i.Dp, D);
            o.Dp = D;
            return products(q8add(i.Qp, o.Qp), gy);
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
            emit(padd(i.P, Hn));
            o.P = padd(i.Hp, Hn);
            o.Hp = Hn;
        };
        /// Two rows: box(o) = P + H1, box(o+1) = Hp + (H1 + H2), and the
        /// pair sum H1 + H2 is the next P (3 vertical adds per 2 rows).
        /// The box state stays in A.
        auto pair_step = [&](int j) {
            const Prod3 H1 = sobel_step(j, A, B);
            emit(padd(A.P, H1));
            const Prod3 H2 = sobel_step(j + 1, B, A);
            A.P = padd(H1, H2);
            emit(padd(A.Hp, A.P));
            A.Hp = H2;
        };
        auto last_step = [&](int j, const State& i, State& o) {
            // product row H clamps to row H-1 at the bottom border
            const Prod3 Hn = sobel_step(j, i, o);
            emit(padd(i.P, (y1 == H) ? i.Hp : Hn));
        };
        int j = 4;
        // 4 rows per iteration on interior strips (loop-carried copies
        // re-aligned once per 4 rows; j % 4 == 0: one chunk check)
        if (!kEdge && GVX_HARRIS_UNROLL >= 4)
            for (; j + 4 < steps; j += 4) {
                if (j % kHarChunk == 0) next_chunk(j / kHarChunk);
                pair_step(j);
                pair_step(j + 2);
            }
        for (; j + 2 < steps; j += 2) {
            if (j % kHarChunk == 0) next_chunk(j / kHarChunk);
            pair_step(j);
        }
        if (j % kHarChunk == 0) next_chunk(j / kHarChunk);
        if (j + 1 < steps) {
            full_step(j, A, B);
            last_step(j + 1, B, A);
        } else {
            last_step(j, A, B);
        }
    };
    // right border: the product at column x + 248 (right neighbour of the
    // strip's last output) or any output column lies past W-1
    if (col_patch || x + kHarCols + 1 > W) body(std::true_type{});
    else body(std::false_type{});
}

// ----------------------------------------------------------------------------
// harris4_kernel: the same computation with 4 columns per lane (pairs
// (c, c+2), (c+1, c+3)), half the per-lane state of harris_kernel, so about
// twice the resident warps.  Strip of 124 output columns: lane L holds
// columns c = x - 2 + 4L .. c + 3; lane 0's first two and lane 31's last two
// columns are halo.  Source rows stream through the same 16-row TMA ring
// (160-byte rows).

constexpr int kH4Cols = 124;
constexpr int kH4SW = 160;

struct Q4p {
    float2 v[2]; // (c, c+2), (c+1, c+3)
};
struct Raw4 {
    float2 v[4]; // (c+i, c+2+i), i = -1 .. 2
};
struct Prod3q {
    Q4p xx, yy, xy;
};
__device__ __forceinline__ Q4p q4add(const Q4p& a, const Q4p& b) { return Q4p{{add2(a.v[0], b.v[0]), add2(a.v[1], b.v[1])}}; }
__device__ __forceinline__ Prod3q padd4(const Prod3q& a, const Prod3q& b) {
    return Prod3q{q4add(a.xx, b.xx), q4add(a.yy, b.yy), q4add(a.xy, b.xy)};
}

template <bool kResp>
__global__ void __launch_bounds__(kHarThreads, GVX_HARRIS4_MINB) harris4_kernel(const __grid_constant__ CUtensorMap map,
                                                                             HarrisParams p) {
    __shared__ alignas(128) uint8_t ring[kHarRing * kH4SW];
    __shared__ uint64_t bar[2];

    const int lane = threadIdx.x;
    // first output column: a multiple of 4; the last strip is pulled left to
    // end at roundup4(W) (overlapping columns are computed twice, identically)
    const int x = max(0, min(static_cast<int>(blockIdx.x) * kH4Cols, ((p.width + 3) & ~3) - kH4Cols));
    const int x_org = ((x - 3) >> 4) << 4;
    const int y0 = p.band.row0 + blockIdx.y * p.th;
    const int y1 = min(y0 + p.th, p.band.row1);
    const int frame = blockIdx.z;
    const int H = p.band.global_h;
    const int W = p.width;
    const int steps = (y1 - y0) + 4;
    const int nchunks = (steps + kHarChunk - 1) / kHarChunk;

    pdl_prologue(p.pdl_wait);
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    __syncwarp();

    auto issue = [&](int k) {
        uint64_t* b = &bar[k & 1];
        mbar_expect_tx(b, kHarChunk * kH4SW);
        tma_load_3d(ring + (k & 1) * kHarChunk * kH4SW, &map, b, x_org / 4, y0 - 2 + kHarChunk * k - p.band.src_row0,
                    frame);
    };
    const bool col_patch = x_org < 0 || x_org + kH4SW > W;
    bool dirty = false;
    auto patch = [&](int k) {
        uint8_t* base = ring + (k & 1) * kHarChunk * kH4SW;
        const int g0 = y0 - 2 + kHarChunk * k;
        const bool rows = g0 < 0 || g0 + kHarChunk > H;
        if (col_patch) {
            const int first = clampi(-x_org, 0, kH4SW - 1), lastc = clampi(W - 1 - x_org, 0, kH4SW - 1);
            for (int r = 0; r < kHarChunk; ++r) {
                uint8_t* row = base + r * kH4SW;
                if (lane < first) row[lane] = row[first];
                for (int j = lastc + 1 + lane; j < kH4SW; j += 32) row[j] = row[lastc];
            }
            __syncwarp();
        }
        if (rows) {
            for (int r = 0; r < kHarChunk; ++r) {
                const int gy = g0 + r;
                if ((gy >= 0 && gy < H) || kHarChunk * k + r >= steps) continue;
                const int v = clampi(gy, 0, H - 1) - (y0 - 2);
                const uint32_t* from = reinterpret_cast<const uint32_t*>(ring + (v % kHarRing) * kH4SW);
                uint32_t* to = reinterpret_cast<uint32_t*>(base + r * kH4SW);
                for (int j = lane; j < kH4SW / 4; j += 32) to[j] = from[j];
            }
            __syncwarp();
        }
        return col_patch || rows;
    };
    auto next_chunk = [&](int k) {
        mbar_wait(&bar[k & 1], (k >> 1) & 1);
        const bool patched = patch(k);
        if (lane == 0 && k + 1 < nchunks) {
            if (dirty) fence_proxy_async_smem();
            issue(k + 1);
        }
        dirty = patched;
    };

    const int c = x - 2 + 4 * lane; // first column of this lane
    const int off = c - x_org;       // ring column (off % 4 == 2)
    const int last = W - 1 - c;      // index of column W-1 among c .. c+3 (when 0..3)
    const bool store_a = lane > 0 && c < W;
    const bool store_b = lane < 31 && c + 2 < W;

    uint8_t* mrow = p.mask + frame * p.mask_fstride + static_cast<int64_t>(y0 - p.band.dst_row0) * p.mask_pitch + c;
    char* rrow = reinterpret_cast<char*>(p.resp) + frame * p.resp_fstride +
                 static_cast<int64_t>(y0 - p.band.dst_row0) * p.resp_pitch;
    const float2 two = f2(2.f, 2.f);

    if (lane == 0) issue(0);
    next_chunk(0);

    auto body = [&](auto edge_tag) {
        constexpr bool kEdge = decltype(edge_tag)::value;
        /// Source row j: pairs (c+i, c+2+i) for i = -1 .. 2 as 2^15 + x.
        auto raw_pairs = [&](int j) {
            const uint8_t* row = ring + (j % kHarRing) * kH4SW + off;
            const uint32_t w0 = *reinterpret_cast<const uint32_t*>(row - 2); // columns c-2 .. c+1
            const uint32_t w1 = *reinterpret_cast<const uint32_t*>(row + 2); // columns c+2 .. c+5
            Raw4 r;
            r.v[0] = f2(magic15_byte(w0, 1), magic15_byte(w0, 3));
            r.v[1] = f2(magic15_byte(w0, 2), magic15_byte(w1, 0));
            r.v[2] = f2(magic15_byte(w0, 3), magic15_byte(w1, 1));
            r.v[3] = f2(magic15_byte(w1, 0), magic15_byte(w1, 2));
            return r;
        };
        auto sobel_d = [&](const Raw4& q) { return Q4p{{sub2(q.v[2], q.v[0]), sub2(q.v[3], q.v[1])}}; };
        auto smooth = [&](const Raw4& q) {
            return Q4p{{fma2(two, q.v[1], add2(q.v[0], q.v[2])), fma2(two, q.v[2], add2(q.v[1], q.v[3]))}};
        };
        /// Columns beyond W-1 take column W-1's value; at the left border the
        /// product at column -1 (lane 0's c+1) takes column 0's (c+2).
        auto clamp_cols = [&](Q4p& q) {
            if (!kEdge) return;
            if (last < 3) {
                float v[4] = {q.v[0].x, q.v[1].x, q.v[0].y, q.v[1].y};
#pragma unroll
                for (int i = 1; i < 4; ++i)
                    if (i > last) v[i] = v[i - 1];
                q.v[0] = f2(v[0], v[2]);
                q.v[1] = f2(v[1], v[3]);
            }
            if (x == 0 && lane == 0) q.v[1].x = q.v[0].y;
        };
        /// Horizontal 3-sums; columns c-1 / c+4 come from the adjacent lanes.
        auto hsum = [&](const Q4p& q) {
            const float L = __shfl_up_sync(0xffffffffu, q.v[1].y, 1); // left lane's c+3 = my c-1
            float R = __shfl_down_sync(0xffffffffu, q.v[0].x, 1);     // right lane's c = my c+4
            if (kEdge) R = last <= 3 ? q.v[1].y : R;
            const float2 sa = add2(q.v[0], q.v[1]);
            return Q4p{{f2(L + sa.x, q.v[1].x + sa.y), f2(sa.x + q.v[0].y, sa.y + R)}};
        };
        auto products = [&](const Q4p& gx, const Q4p& gy) {
            Q4p xx{{mul2(gx.v[0], gx.v[0]), mul2(gx.v[1], gx.v[1])}};
            Q4p yy{{mul2(gy.v[0], gy.v[0]), mul2(gy.v[1], gy.v[1])}};
            Q4p xy{{mul2(gx.v[0], gy.v[0]), mul2(gx.v[1], gy.v[1])}};
            clamp_cols(xx);
            clamp_cols(yy);
            clamp_cols(xy);
            return Prod3q{hsum(xx), hsum(yy), hsum(xy)};
        };
        auto emit = [&](const Prod3q& V) {
            uint32_t ma = 0, mb = 0; // bytes (c, c+1) and (c+2, c+3)
            float rv[4];             // columns c .. c+3
            if constexpr (kResp) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    rv[i] = exact_response(V.xx.v[i].x, V.yy.v[i].x, V.xy.v[i].x, p.k);
                    rv[i + 2] = exact_response(V.xx.v[i].y, V.yy.v[i].y, V.xy.v[i].y, p.k);
                    ma |= (static_cast<double>(rv[i]) > p.threshold ? 255u : 0u) << (8 * i);
                    mb |= (static_cast<double>(rv[i + 2]) > p.threshold ? 255u : 0u) << (8 * i);
                }
            } else {
                const float2 kk = f2(p.kpos, p.kpos), t81 = f2(p.t81, p.t81);
                const float2 ctt = f2(p.c_tt, p.c_tt), c0 = f2(p.c0, p.c0);
                float2 nd[2], e[2];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float2 tr = add2(V.xx.v[i], V.yy.v[i]);
                    const float2 tt = mul2(tr, tr);
                    const float2 w = fma2(V.xy.v[i], V.xy.v[i], t81);
                    const float2 ndet = fma2(f2(-V.xx.v[i].x, -V.xx.v[i].y), V.yy.v[i], w);
                    nd[i] = fma2(kk, tt, ndet);
                    e[i] = fma2(ctt, tt, c0);
                }
                bool unsure = false;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    unsure |= !(fabsf(nd[i].x) > e[i].x);
                    unsure |= !(fabsf(nd[i].y) > e[i].y);
                }
                // mask byte = sign of nd replicated (nd < 0 <=> resp > T)
                ma = sign_bytes(nd[0].x, nd[1].x);
                mb = sign_bytes(nd[0].y, nd[1].y);
                if (__any_sync(0xffffffffu, unsure)) {
                    unsigned ub = 0;
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        ub |= (fabsf(nd[i].x) > e[i].x ? 0u : 1u) << i;
                        ub |= (fabsf(nd[i].y) > e[i].y ? 0u : 1u) << (i + 2);
                    }
                    if (ub) {
                        float buf[12];
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            buf[i] = V.xx.v[i].x, buf[i + 2] = V.xx.v[i].y;
                            buf[4 + i] = V.yy.v[i].x, buf[6 + i] = V.yy.v[i].y;
                            buf[8 + i] = V.xy.v[i].x, buf[10 + i] = V.xy.v[i].y;
                        }
#pragma unroll 1
                        while (ub) {
                            const int i = __ffs(ub) - 1;
                            ub &= ub - 1;
                            const bool on =
                                static_cast<double>(exact_response(buf[i], buf[4 + i], buf[8 + i], p.k)) > p.threshold;
                            const int sh = 8 * (i & 1);
                            const uint32_t bit = (on ? 255u : 0u) << sh, keep = ~(255u << sh);
                            if (i < 2) ma = (ma & keep) | bit;
                            else mb = (mb & keep) | bit;
                        }
                    }
                }
                (void)rv;
            }
            uint8_t* mp = mrow;
            mrow += p.mask_pitch;
            if (!kEdge || c + 3 < W) {
                if (store_a) *reinterpret_cast<uint16_t*>(mp) = static_cast<uint16_t>(ma);
                if (store_b) *reinterpret_cast<uint16_t*>(mp + 2) = static_cast<uint16_t>(mb);
            } else {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    if (store_a && c + i < W) mp[i] = static_cast<uint8_t>(ma >> (8 * i));
                    if (store_b && c + 2 + i < W) mp[2 + i] = static_cast<uint8_t>(mb >> (8 * i));
                }
            }
            if constexpr (kResp) {
                float* rp = reinterpret_cast<float*>(rrow) + c;
                rrow += p.resp_pitch;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    if (store_a && c + i < W) rp[i] = rv[i];
                    if (store_b && c + 2 + i < W) rp[2 + i] = rv[2 + i];
                }
            }
        };

        struct State {
            Q4p Dp, Qp; // D(r-1), Q(r-1)
            Q4p S;      // smoothing S of the source row this copy last consumed
            Prod3q P, Hp;
        };
        State A, B;
        {
            const Raw4 r0 = raw_pairs(0), r1 = raw_pairs(1);
            B.S = smooth(r0);
            A.S = smooth(r1);
            const Q4p D0 = sobel_d(r0), D1 = sobel_d(r1);
            A.Qp = q4add(D0, D1);
            A.Dp = D1;
        }
        auto sobel_step = [&](int j, const State& i, State& o) {
            const Raw4 q = raw_pairs(j);
            const Q4p D = sobel_d(q);
            const Q4p S = smooth(q);
            const Q4p gy{{sub2(S.v[0], o.S.v[0]), sub2(S.v[1], o.S.v[1])}};
            o.S = S;
            o.Qp = q4add(i.Dp, D);
            o.Dp = D;
            return products(q4add(i.Qp, o.Qp), gy);
        };
        {
            const Prod3q H1 = sobel_step(2, A, B);
            const Prod3q H2 = sobel_step(3, B, A);
            A.P = padd4(y0 == 0 ? H2 : H1, H2);
            A.Hp = H2;
        }
        auto full_step = [&](int j, const State& i, State& o) {
            const Prod3q Hn = sobel_step(j, i, o);
            emit(padd4(i.P, Hn));
            o.P = padd4(i.Hp, Hn);
            o.Hp = Hn;
        };
        auto last_step = [&](int j, const State& i, State& o) {
            const Prod3q Hn = sobel_step(j, i, o);
            emit(padd4(i.P, (y1 == H) ? i.Hp : Hn));
        };
        auto pair_step = [&](int j) {
            const Prod3q H1 = sobel_step(j, A, B);
            emit(padd4(A.P, H1));
            const Prod3q H2 = sobel_step(j + 1, B, A);
            A.P = padd4(H1, H2);
            emit(padd4(A.Hp, A.P));
            A.Hp = H2;
        };
        int j = 4;
        if (!kEdge && GVX_HARRIS4_UNROLL >= 4)
            for (; j + 4 < steps; j += 4) {
                if (j % kHarChunk == 0) next_chunk(j / kHarChunk);
                pair_step(j);
                pair_step(j + 2);
            }
        for (; j + 2 < steps; j += 2) {
            if (j % kHarChunk == 0) next_chunk(j / kHarChunk);
            pair_step(j);
        }
        if (j % kHarChunk == 0) next_chunk(j / kHarChunk);
        if (j + 1 < steps) {
            full_step(j, A, B);
            last_step(j + 1, B, A);
        } else {
            last_step(j, A, B);
        }
    };
    if (col_patch || x + kH4Cols + 1 > W) body(std::true_type{});
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
    // 4 columns per lane (harris4_kernel, 94 registers, ~21 warps / SM) unless
    // GVX_HARRIS8 asks for the 8-column kernel (164 registers, 12 warps / SM):
    // measured 926 vs 886 Gpx/s batched, 754 vs 585 one frame per launch
    static const bool four = std::getenv("GVX_HARRIS8") == nullptr;
    const int cols = four ? kH4Cols : kHarCols, sw = four ? kH4SW : kHarSW;
    void* fn = four ? (a->response.data ? reinterpret_cast<void*>(&harris4_kernel<true>)
                                        : reinterpret_cast<void*>(&harris4_kernel<false>))
                    : (a->response.data ? reinterpret_cast<void*>(&harris_kernel<true>)
                                        : reinterpret_cast<void*>(&harris_kernel<false>));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kHarThreads, 0);
    const long long strips = static_cast<long long>(frames) * ((s.width + cols - 1) / cols);
    p.th = balanced_tile_rows(strips, rows, static_cast<long long>(per_sm > 0 ? per_sm : 1) * ctx->sm_count,
                              kHarTHMax, 4);
    if (const char* e = std::getenv("GVX_HARRIS_TH")) p.th = std::max(8, std::atoi(e)); // tuning experiments
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, sw, kHarChunk)) return rc;
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
    p.kpos = static_cast<float>(a->k);
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
    p.c_tt = static_cast<float>((c_tt + c_tr / (2.0 * a_tr)) * 1.001);
    p.c0 = static_cast<float>((c_0 + c_tr * a_tr / 2.0) * 1.001 + 1.0);
    dim3 grid((s.width + cols - 1) / cols, (rows + p.th - 1) / p.th, frames);
    // rows read (band +- 2, within the slab) and written (band rows)
    const int b0 = a->band.row0, b1 = a->band.row1;
    const gvxb_range r[1] = {rows_range(s, b0 - 2 - a->band.src_row0, b1 - b0 + 4)};
    const gvxb_range w[2] = {rows_range(a->mask, b0 - a->band.dst_row0, b1 - b0),
                             rows_range(a->response, b0 - a->band.dst_row0, b1 - b0)};
    p.pdl_wait = pdl_must_wait(ctx, r, 1, w, 2);
    void* args[] = {&map, &p};
    return launch_tracked(ctx, fn, grid, dim3(kHarThreads), args, 0, r, 1, w, 2, "harris kernel");
}
