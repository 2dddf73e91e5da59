// K1 v4 — fused Gaussian3x3 -> Sobel3x3 -> {gx, gy, Magnitude} (U8 -> S16)
// in the layout of the Harris kernel: one warp per CTA, 8 columns per lane,
// source rows streamed through a TMA row ring, long row bands.
//
// Reference semantics, exactly as edge.cu:
//   gaussian3x3  floor((s + 8) / 16), s <= 4080   (ref:src/registry.cpp:722-746)
//   sobel_x/y    sat_S16(sum(mask * win)), |v| <= 1020 (ref:src/registry.cpp:748-784)
//   magnitude    sat_S16(llround(sqrt(gx^2 + gy^2))) (ref:src/registry.cpp:555-575)
//   Clamp of the intermediate: the Gaussian at an out-of-image position is
//   the Gaussian of the clamped position (ref:src/execute.cpp:242-245).
//
// The work is split across the SM sub-partition's two arithmetic pipes: the
// Gaussian runs as 16-bit SWAR integer arithmetic on the ALU pipe (PRMT /
// LEA / IADD3 / LOP3, two columns per 32-bit register), the Sobel and the
// magnitude as packed FP32 (FFMA2 / FADD2 / FMUL2) on the FMA pipe.
//
// Layout: a strip of 248 output columns per warp; lane L holds columns
// c = x - 4 + 8L .. c + 7; only lane 0's first half and lane 31's second
// half are halo.  Per source row j (virtual row j <-> global row y0 - 2 + j):
//   h(j)        horizontal 1-2-1 of the source bytes as SWAR words of the
//               column pairs E1 = (c, c+2), O1 = (c+1, c+3), E2 = (c+4, c+6),
//               O2 = (c+5, c+7) (byte permutes of the ring words)
//   G(j-1)      = (h(j-2) + 2 h(j-1) + h(j) + 8) & ~15 = 16 floor((S + 8) / 16)
//               (running sums R = h(j-1) + h(j)); each 16-bit lane becomes the
//               float 2^23 + 16 g by one byte permute, as pairs (c+i, c+4+i)
//   gx(j-2)     = Q(j-2) + Q(j-1), Q(m) = D(m-1) + D(m), D = G(x+1) - G(x-1)
//   gy(j-2)     = horizontal 1-2-1 of G(j-1) - G(j-3) (the 2^23 cancels)
// so output row j - 4 is emitted at step j, gx and gy scaled by 16.  Every
// quantity is an integer times 16 below 2^24 (squares: times 256 below
// 2^30 with <= 21 significant bits): exact in fp32.
#include "packed.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace gvxd {

constexpr int kE8Threads = 32;  // one warp per CTA
constexpr int kE8Cols = 248;    // output columns per strip
constexpr int kE8SW = 288;      // ring row bytes: image columns [x_org, x_org + 288)
constexpr int kE8Chunk = 16;    // rows per TMA chunk
constexpr int kE8Ring = 2 * kE8Chunk;
constexpr int kE8THMax = 256;   // band rows: with overlapped launches taller bands win (halo rows amortised; measured 64 -> 256: +1.7% on 16K^2)
constexpr int kE8THSerial = 64; // band rows when the launch waits for its predecessor: the grid's tail is exposed, so
                                // shorter bands balance better (measured 16384^2: 211 -> 192 us, 64 x 1080p: +6%)

struct E8Plane {
    int16_t* data;
    int64_t pitch, frame_stride; // bytes
};

struct Edge8Params {
    int width;
    int th;
    int pdl_wait; // the previous grid on the stream may have written what this one touches
    Band band;
    E8Plane gx, gy, mag;
};

struct P8 {
    float2 v[4]; // (c+i, c+4+i)
};
/// Six pairs for i = -1 .. 4 at v[i + 1]: columns (c+i, c+4+i).
struct P12 {
    float2 v[6];
};
/// A Gaussian row around the lane: its 8 columns and the two neighbour
/// pairs lp = (c-1, c+3), rp = (c+4, c+8), so every 3-tap step is packed.
struct GRow {
    P8 g;
    float2 lp, rp;
};

__device__ __forceinline__ float e8_sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

/// round(sqrt(n)) half away from zero, in magic form 2^23 + k (low 16 bits
/// = k), from n64 = 256 n + 64 = 64 (4 n + 1) (gx, gy carry a factor 16;
/// the caller folds in the 64).  s = sqrt~(n64) = 16 sqrt(n + 1/4) (1 + e),
/// |e| < 2^-21, and sqrt(n + 1/4) lies in [k* - 1/2, k* + 1/2] for the
/// rounded root k*, so k0 = floor(s / 16) (one FFMA2 rounding down into the
/// magic range) is k* or k* - 1, and k* = k0 + (n > k0 (k0 + 1)).  With
/// v = 16 k0 + 8, u = v^2 - n64 = 256 (k0 (k0 + 1) - n) is exact (multiples
/// of 64 below 2^30) and negative exactly when the increment applies.  The
/// increment is one more packed FMA rounding upward: km - u 2^-21 with
/// |u| 2^-21 < 1 rounds to km + 1 for u < 0 and to km otherwise (ulp(km) = 1).
__device__ __forceinline__ float2 e8_round_sqrt16(float2 n64) {
    const float2 s = f2(e8_sqrt_approx(n64.x), e8_sqrt_approx(n64.y));
    const float2 km = __ffma2_rd(s, f2(0.0625f, 0.0625f), f2(8388608.f, 8388608.f)); // 2^23 + k0
    const float2 v = __ffma2_rn(km, f2(16.f, 16.f), f2(-134217720.f, -134217720.f)); // 16 k0 + 8 (2^27 - 8 is exact)
    const float2 u = __ffma2_rn(v, v, f2(-n64.x, -n64.y));
    return __ffma2_ru(u, f2(-4.76837158203125e-07f, -4.76837158203125e-07f), km); // 2^23 + k*
}

/// 16-bit lane `hi` of a SWAR word as the float 2^23 + lane (one permute).
__device__ __forceinline__ float e8_lane(uint32_t w, int hi) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, hi ? 0x7632u : 0x7610u));
}

/// 16 x (integer-valued floats |v| < 2^18) as two int16 v in a u32.
__device__ __forceinline__ uint32_t e8_pack16(float lo, float hi) {
    const float m = 12582912.f;
    return __byte_perm(__float_as_uint(fmaf(lo, 0.0625f, m)), __float_as_uint(fmaf(hi, 0.0625f, m)), 0x5410);
}
/// Magic-form values (1.5*2^23 + v) as two int16 in a u32.
__device__ __forceinline__ uint32_t e8_pack_magic(float lo, float hi) {
    return __byte_perm(__float_as_uint(lo), __float_as_uint(hi), 0x5410);
}

#ifndef GVX_EDGE8_UNROLL
#define GVX_EDGE8_UNROLL 4 // rows per loop iteration of interior strips (2 or 4)
#endif
template <bool kGx, bool kGy, bool kMag>
#ifndef GVX_EDGE8_MINB
#define GVX_EDGE8_MINB 1
#endif
__global__ void __launch_bounds__(kE8Threads, GVX_EDGE8_MINB) edge8_kernel(const __grid_constant__ CUtensorMap map, Edge8Params p) {
    __shared__ alignas(128) uint8_t ring[kE8Ring * kE8SW];
    __shared__ uint64_t bar[2];

    const int lane = threadIdx.x;
    const int x = max(0, min(static_cast<int>(blockIdx.x) * kE8Cols, ((p.width + 7) & ~7) - kE8Cols));
    const int x_org = ((x - 5) >> 4) << 4; // ring column 0 (16-byte aligned TMA origin)
    const int y0 = p.band.row0 + blockIdx.y * p.th;
    const int y1 = min(y0 + p.th, p.band.row1);
    const int frame = blockIdx.z;
    const int H = p.band.global_h;
    const int W = p.width;
    const int steps = (y1 - y0) + 4;
    const int nchunks = (steps + kE8Chunk - 1) / kE8Chunk;

    pdl_prologue(p.pdl_wait);
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    __syncwarp();

    auto issue = [&](int k) {
        uint64_t* b = &bar[k & 1];
        mbar_expect_tx(b, kE8Chunk * kE8SW);
        tma_load_3d(ring + (k & 1) * kE8Chunk * kE8SW, &map, b, x_org / 4, y0 - 2 + kE8Chunk * k - p.band.src_row0,
                    frame);
    };
    const bool col_patch = x_org < 0 || x_org + kE8SW > W;
    bool dirty = false;
    auto patch = [&](int k) {
        uint8_t* base = ring + (k & 1) * kE8Chunk * kE8SW;
        const int g0 = y0 - 2 + kE8Chunk * k;
        const bool rows = g0 < 0 || g0 + kE8Chunk > H;
        if (col_patch) {
            const int first = clampi(-x_org, 0, kE8SW - 1), lastc = clampi(W - 1 - x_org, 0, kE8SW - 1);
            for (int r = 0; r < kE8Chunk; ++r) {
                uint8_t* row = base + r * kE8SW;
                if (lane < first) row[lane] = row[first];
                for (int j = lastc + 1 + lane; j < kE8SW; j += 32) row[j] = row[lastc];
            }
            __syncwarp();
        }
        if (rows) {
            for (int r = 0; r < kE8Chunk; ++r) {
                const int gy = g0 + r;
                if ((gy >= 0 && gy < H) || kE8Chunk * k + r >= steps) continue;
                const int v = clampi(gy, 0, H - 1) - (y0 - 2);
                const uint32_t* from = reinterpret_cast<const uint32_t*>(ring + (v % kE8Ring) * kE8SW);
                uint32_t* to = reinterpret_cast<uint32_t*>(base + r * kE8SW);
                for (int j = lane; j < kE8SW / 4; j += 32) to[j] = from[j];
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

    const int c = x - 4 + 8 * lane;
    const int off = c - x_org; // 4 <= off, off % 8 == 4
    const int last = W - 1 - c;
    const bool store_a = lane > 0 && c < W;
    const bool store_b = lane < 31 && c + 4 < W;
    auto out_row = [&](const E8Plane& o) {
        return reinterpret_cast<char*>(o.data) + frame * o.frame_stride +
               static_cast<int64_t>(y0 - p.band.dst_row0) * o.pitch + 2 * static_cast<int64_t>(c);
    };
    char* pgx = kGx ? out_row(p.gx) : nullptr;
    char* pgy = kGy ? out_row(p.gy) : nullptr;
    char* pmag = kMag ? out_row(p.mag) : nullptr;

    if (lane == 0) issue(0);
    next_chunk(0);

    auto body = [&](auto edge_tag) {
        constexpr bool kEdge = decltype(edge_tag)::value;
        /// Horizontal 1-2-1 of source row j as SWAR words {E1, O1, E2, O2}
        /// (16-bit lanes, sums <= 1020).  L / R are the neighbour-column pairs
        /// built by permutes with a zero lane from the unpacked words.
        auto hsum = [&](int j, uint32_t* h) {
            const uint8_t* row = ring + (j % kE8Ring) * kE8SW + off;
            const uint2 lo = *reinterpret_cast<const uint2*>(row - 4), hi = *reinterpret_cast<const uint2*>(row + 4);
            const uint32_t E1 = __byte_perm(lo.y, 0, 0x4240), O1 = __byte_perm(lo.y, 0, 0x4341);
            const uint32_t E2 = __byte_perm(hi.x, 0, 0x4240), O2 = __byte_perm(hi.x, 0, 0x4341);
            const uint32_t LE1 = __byte_perm(lo.x, O1, 0x5453); // (c-1, c+1)
            const uint32_t RO1 = __byte_perm(E1, hi.x, 0x1412); // (c+2, c+4)
            const uint32_t LE2 = __byte_perm(O1, O2, 0x1412);   // (c+3, c+5)
            const uint32_t RO2 = __byte_perm(E2, hi.y, 0x1412); // (c+6, c+8)
            h[0] = (E1 << 1) + LE1 + O1;
            h[1] = (O1 << 1) + E1 + RO1;
            h[2] = (E2 << 1) + LE2 + O2;
            h[3] = (O2 << 1) + E2 + RO2;
        };
        const float2 two = f2(2.f, 2.f);
        /// Gaussian columns beyond W-1 take column W-1's value; column -1
        /// (lane 0's A3 in the first strip) takes column 0's (B0).
        auto clamp_cols = [&](P8& g) {
            if (!kEdge) return;
            if (last < 7) {
                float v[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    v[i] = g.v[i].x;
                    v[i + 4] = g.v[i].y;
                }
#pragma unroll
                for (int i = 1; i < 8; ++i)
                    if (i > last) v[i] = v[i - 1];
#pragma unroll
                for (int i = 0; i < 4; ++i) g.v[i] = f2(v[i], v[i + 4]);
            }
            if (x == 0 && lane == 0) g.v[3].x = g.v[0].y;
        };
        /// Gaussian row with columns c-1 / c+8 from the neighbour lanes
        /// (clamped at the image border).
        auto neighbourhood = [&](const P8& g) {
            const float L = __shfl_up_sync(0xffffffffu, g.v[3].y, 1);
            float R = __shfl_down_sync(0xffffffffu, g.v[0].x, 1);
            if (kEdge) R = last <= 7 ? g.v[3].y : R;
            return GRow{g, f2(L, g.v[3].x), f2(g.v[0].y, R)};
        };
        auto emit = [&](const P8& gx, const P8& gy) {
            const bool full = !kEdge || c + 7 < W;
            auto put = [&](char* base, uint32_t a01, uint32_t a23, uint32_t b01, uint32_t b23) {
                if (full) {
                    if (store_a) *reinterpret_cast<uint2*>(base) = make_uint2(a01, a23);
                    if (store_b) *reinterpret_cast<uint2*>(base + 8) = make_uint2(b01, b23);
                } else {
                    const uint32_t w[4] = {a01, a23, b01, b23};
                    int16_t* q = reinterpret_cast<int16_t*>(base);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const bool mine = i < 4 ? store_a : store_b;
                        if (mine && c + i < W) q[i] = static_cast<int16_t>(w[i >> 1] >> (16 * (i & 1)));
                    }
                }
            };
            if (kGx) {
                put(pgx, e8_pack16(gx.v[0].x, gx.v[1].x), e8_pack16(gx.v[2].x, gx.v[3].x), e8_pack16(gx.v[0].y, gx.v[1].y),
                    e8_pack16(gx.v[2].y, gx.v[3].y));
                pgx += p.gx.pitch;
            }
            if (kGy) {
                put(pgy, e8_pack16(gy.v[0].x, gy.v[1].x), e8_pack16(gy.v[2].x, gy.v[3].x), e8_pack16(gy.v[0].y, gy.v[1].y),
                    e8_pack16(gy.v[2].y, gy.v[3].y));
                pgy += p.gy.pitch;
            }
            if (kMag) {
                float2 m[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) m[i] = e8_round_sqrt16(fma2(gx.v[i], gx.v[i], fma2(gy.v[i], gy.v[i], f2(64.f, 64.f))));
                put(pmag, e8_pack_magic(m[0].x, m[1].x), e8_pack_magic(m[2].x, m[3].x), e8_pack_magic(m[0].y, m[1].y),
                    e8_pack_magic(m[2].y, m[3].y));
                pmag += p.mag.pitch;
            }
        };

        // State of the running sums; two alternating copies (A, B) so the
        // 2x-unrolled loop renames instead of moving registers.
        struct State {
            uint32_t hp[4], rp[4]; // h(j-1), h(j-2) + h(j-1) (SWAR)
            P8 Dp, Qp;             // D(m), Q(m) of the newest Gaussian row
            P8 Hn;                 // H of the Gaussian row this copy last produced
        };
        State A, B;
        /// Source row j -> Gaussian row j-1 (2^23 + 16 g, clamped columns).
        auto gauss_step = [&](int j, const State& i, State& o) {
            uint32_t h[4], g16[4];
            hsum(j, h);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                o.rp[t] = i.hp[t] + h[t];
                g16[t] = (i.rp[t] + o.rp[t] + 0x00080008u) & 0xFFF0FFF0u;
                o.hp[t] = h[t];
            }
            P8 g; // pairs (c+i, c+4+i): E1 = (c, c+2), O1 = (c+1, c+3), E2, O2 = +4
            g.v[0] = f2(e8_lane(g16[0], 0), e8_lane(g16[2], 0));
            g.v[1] = f2(e8_lane(g16[1], 0), e8_lane(g16[3], 0));
            g.v[2] = f2(e8_lane(g16[0], 1), e8_lane(g16[2], 1));
            g.v[3] = f2(e8_lane(g16[1], 1), e8_lane(g16[3], 1));
            clamp_cols(g);
            return neighbourhood(g);
        };
        /// D = G(x+1) - G(x-1) for the lane's 8 columns.
        auto diff = [&](const GRow& n) {
            P8 d;
            d.v[0] = sub2(n.g.v[1], n.lp);
            d.v[1] = sub2(n.g.v[2], n.g.v[0]);
            d.v[2] = sub2(n.g.v[3], n.g.v[1]);
            d.v[3] = sub2(n.rp, n.g.v[2]);
            return d;
        };
        /// Horizontal 1-2-1 of a Gaussian row: gy(r) = H(r+1) - H(r-1).
        auto hsmooth = [&](const GRow& n) {
            P8 h;
            h.v[0] = fma2(two, n.g.v[0], add2(n.lp, n.g.v[1]));
            h.v[1] = fma2(two, n.g.v[1], add2(n.g.v[0], n.g.v[2]));
            h.v[2] = fma2(two, n.g.v[2], add2(n.g.v[1], n.g.v[3]));
            h.v[3] = fma2(two, n.g.v[3], add2(n.g.v[2], n.rp));
            return h;
        };
        // prologue: h rows 0, 1; Gaussian rows y0-1 (j = 2) and y0 (j = 3)
        {
            uint32_t h0[4];
            hsum(0, h0);
            hsum(1, A.hp);
#pragma unroll
            for (int t = 0; t < 4; ++t) A.rp[t] = h0[t] + A.hp[t];
        }
        GRow G1 = gauss_step(2, A, B); // Gaussian row y0-1
        GRow G2 = gauss_step(3, B, A); // Gaussian row y0
        if (y0 == 0) G1 = G2;          // Gaussian row -1 clamps to row 0
        {
            const P8 D1 = diff(G1), D2 = diff(G2);
#pragma unroll
            for (int t = 0; t < 4; ++t) A.Qp.v[t] = add2(D1.v[t], D2.v[t]);
            A.Dp = D2;
            A.Hn = hsmooth(G2); // newest row
            B.Hn = hsmooth(G1); // the copy read at the next step holds the row two back
        }
        /// Step j: Gaussian row j-1 -> Sobel / outputs of row j-4 (global).
        /// `bottom`: Gaussian row j-1 is row H, which clamps to row H-1.
        auto full_step = [&](int j, State& i, State& o, bool bottom) {
            const GRow Gn = gauss_step(j, i, o);
            P8 D = diff(Gn), Hn = hsmooth(Gn);
            if (bottom) D = i.Dp, Hn = i.Hn; // Gaussian row H clamps to row H-1
            P8 Q, gx, gy;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                Q.v[t] = add2(i.Dp.v[t], D.v[t]);
                gx.v[t] = add2(i.Qp.v[t], Q.v[t]);
                gy.v[t] = sub2(Hn.v[t], o.Hn.v[t]); // o.Hn = H of Gaussian row j-3
            }
            o.Qp = Q;
            o.Dp = D;
            o.Hn = Hn;
            emit(gx, gy);
        };
        int j = 4;
        // 4 rows per iteration (j % 4 == 0: one chunk check per iteration;
        // the state's loop-carried copies are re-aligned once per 4 rows)
        // (interior strips only: the border variant, with its column clamps,
        // runs faster 2x-unrolled)
        if (!kEdge && GVX_EDGE8_UNROLL >= 4)
        for (; j + 4 < steps; j += 4) {
            if (j % kE8Chunk == 0) next_chunk(j / kE8Chunk);
            full_step(j, A, B, false);
            full_step(j + 1, B, A, false);
            full_step(j + 2, A, B, false);
            full_step(j + 3, B, A, false);
        }
        for (; j + 2 < steps; j += 2) {
            if (j % kE8Chunk == 0) next_chunk(j / kE8Chunk);
            full_step(j, A, B, false);
            full_step(j + 1, B, A, false);
        }
        if (j % kE8Chunk == 0) next_chunk(j / kE8Chunk);
        const bool bot = y1 == H;
        if (j + 1 < steps) {
            full_step(j, A, B, false);
            full_step(j + 1, B, A, bot);
        } else {
            full_step(j, A, B, bot);
        }
    };
    if (col_patch || x + kE8Cols + 1 > W) body(std::true_type{});
    else body(std::false_type{});
}

template <bool X, bool Y>
void* pick_e8(bool om) {
    return om ? reinterpret_cast<void*>(&edge8_kernel<X, Y, true>) : reinterpret_cast<void*>(&edge8_kernel<X, Y, false>);
}

} // namespace gvxd

using namespace gvxd;

namespace gvxb_impl {

/// gvxb_edge's Gaussian variants (called from edge.cu).
int edge8_launch(gvxb_ctx ctx, const gvxb_edge_args* a) {
    const gvxb_image& s = a->src;
    const bool ox = a->gx.data, oy = a->gy.data, om = a->mag.data;
    void* fn = ox ? (oy ? pick_e8<true, true>(om) : pick_e8<true, false>(om))
                  : (oy ? pick_e8<false, true>(om) : pick_e8<false, false>(om));
    const int rows = a->band.row1 - a->band.row0;
    const int frames = s.frames > 0 ? s.frames : 1;
#ifndef GVX_EDGE8_CARVEOUT
#define GVX_EDGE8_CARVEOUT 1
#endif
    static bool carveout = !GVX_EDGE8_CARVEOUT; // one-warp CTAs: shared memory must not cap residency
    if (!carveout) {
        for (bool X : {false, true})
            for (bool Y : {false, true})
                for (bool M : {false, true})
                    cudaFuncSetAttribute(X ? (Y ? pick_e8<true, true>(M) : pick_e8<true, false>(M))
                                           : (Y ? pick_e8<false, true>(M) : pick_e8<false, false>(M)),
                                         cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
        carveout = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kE8Threads, 0);
    const long long strips = static_cast<long long>(frames) * ((s.width + kE8Cols - 1) / kE8Cols);
    Edge8Params p;
    // the rows this launch reads (band rows +- 2, clipped to the slab) and
    // writes: bands of one buffer on disjoint rows are independent launches
    const int b0 = a->band.row0, b1 = a->band.row1;
    const gvxb_range r[1] = {rows_range(s, b0 - 2 - a->band.src_row0, b1 - b0 + 4)};
    const gvxb_range w[3] = {rows_range(a->gx, b0 - a->band.dst_row0, b1 - b0),
                             rows_range(a->gy, b0 - a->band.dst_row0, b1 - b0),
                             rows_range(a->mag, b0 - a->band.dst_row0, b1 - b0)};
    const int th_max = launch_overlaps(ctx, r, 1, w, 3) ? kE8THMax : kE8THSerial;
    p.th = balanced_tile_rows(strips, rows, static_cast<long long>(per_sm > 0 ? per_sm : 1) * ctx->sm_count, th_max, 4);
    if (const char* e = std::getenv("GVX_EDGE8_TH")) p.th = std::max(8, std::atoi(e)); // tuning experiments
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, kE8SW, kE8Chunk)) return rc;
    p.width = s.width;
    p.band = Band{a->band.row0, a->band.row1, a->band.global_h, a->band.src_row0, a->band.dst_row0};
    auto plane = [](const gvxb_image& img) {
        E8Plane o;
        o.data = static_cast<int16_t*>(img.data);
        o.pitch = img.pitch;
        o.frame_stride = img.frames > 1 ? img.frame_stride : img.pitch * img.height;
        return o;
    };
    p.gx = plane(a->gx);
    p.gy = plane(a->gy);
    p.mag = plane(a->mag);
    dim3 grid((s.width + kE8Cols - 1) / kE8Cols, (rows + p.th - 1) / p.th, frames);
    p.pdl_wait = pdl_must_wait(ctx, r, 1, w, 3);
    void* args[] = {&map, &p};
    return launch_tracked(ctx, fn, grid, dim3(kE8Threads), args, 0, r, 1, w, 3, "edge8 kernel");
}

} // namespace gvxb_impl
