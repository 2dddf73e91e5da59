// K2 — fused Harris corner graph (U8 -> U8 mask), one pass.
//
// Graph (SURVEY.md §8a "Harris graph definition"): Sobel3x3 -> Multiply
// (gx*gx, gy*gy, gx*gy -> S32) -> Box3x3 (S32) -> user point
// HarrisResponse F32((Sxx*Syy - Sxy^2) - k*(Sxx+Syy)^2) -> user point
// ThresholdF32 sat_U8(resp > T ? 255 : 0).
// Exactness:
//   Sobel |v| <= 1020, products <= 1020^2 (no S32 saturation),
//   Box3x3 post sat_S32(llround(s * (1/9.0))) == round_half_away(s / 9)
//   for |s| <= 9*1020^2 (the double product error < 3e-10 is far below the
//   1/18 distance of s/9 to any half-integer; ref:src/registry.cpp:703-720),
//   response in int64 + IEEE double exactly as the reference evaluates the
//   expression (int64 products, double multiply/subtract, float rounding;
//   ref:src/expr.cpp:351-371), threshold compares double(float(resp)) > T.
//   => bit-exact mask (and response when stored).
//   Clamp of the intermediates: products at out-of-image positions take the
//   value of the clamped position (the Box window clamps into the
//   materialised product image, ref:src/execute.cpp:242-245).
//
// Layout: CTA = 128 threads, tile 512 x 32 outputs; each thread owns 4
// columns and streams rows with 3-row register rings for the separable Sobel
// terms and the horizontal box sums.
#include "tile.cuh"

namespace gvxd {

constexpr int kHarThreads = 128;
constexpr int kHarTW = 4 * kHarThreads;
constexpr int kHarTH = 32;
constexpr int kHarSW = kHarTW + 64; // columns [x0 - 32, x0 + 544)
constexpr int kHarSH = kHarTH + 4;  // rows [y0 - 2, y0 + 34)
constexpr int kHarBox = 192;

struct HarrisParams {
    int width;
    Band band;
    uint8_t* mask;
    int64_t mask_pitch, mask_fstride;
    float* resp;
    int64_t resp_pitch, resp_fstride;
    double k;
    double threshold;
};

__device__ __forceinline__ void fetch8h(const uint8_t* row, int off, int (&a)[8]) {
    const uint32_t wl = lds32(row, off - 4), wc = lds32(row, off), wr = lds32(row, off + 4);
    a[0] = byte_of(wl, 2);
    a[1] = byte_of(wl, 3);
#pragma unroll
    for (int k = 0; k < 4; ++k) a[2 + k] = byte_of(wc, k);
    a[6] = byte_of(wr, 0);
    a[7] = byte_of(wr, 1);
}

__device__ __forceinline__ int box_round(int s) { return round_div_away(s, 9); }

template <bool kResp>
__global__ void __launch_bounds__(kHarThreads) harris_kernel(const __grid_constant__ CUtensorMap map,
                                                             HarrisParams p) {
    __shared__ alignas(128) uint8_t tile[kHarSH * kHarSW];
    __shared__ uint64_t bar;

    const int x0 = blockIdx.x * kHarTW;
    const int y0 = p.band.row0 + blockIdx.y * kHarTH;
    const int y1 = min(y0 + kHarTH, p.band.row1);
    const int frame = blockIdx.z;
    const int H = p.band.global_h;

    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    stage_tile_u8<kHarSW, kHarSH>(tile, &map, &bar, x0 - 32, y0 - 2, frame, p.width, p.band);

    const int c = x0 + 4 * static_cast<int>(threadIdx.x);
    if (c >= p.width) return;
    const int off = 4 * static_cast<int>(threadIdx.x) + 32;
    const int klo = c == 0 ? 0 : -1;              // product column c-1 clamps to c
    const int khi = min(4, p.width - 1 - c);      // last in-image product slot offset

    // separable Sobel terms per source row, columns c-1 .. c+4
    int dA[6], dB[6], dC[6]; // D(k) = in(k+1) - in(k-1)
    int sA[6], sB[6], sC[6]; // S(k) = in(k-1) + 2 in(k) + in(k+1)
    // horizontal box sums of the products per product row, columns c .. c+3
    int xA[4], xB[4], xC[4];
    int yA[4], yB[4], yC[4];
    int zA[4], zB[4], zC[4];

    uint8_t* mrow_base = p.mask + frame * p.mask_fstride;
    char* rrow_base = reinterpret_cast<char*>(p.resp) + frame * p.resp_fstride;

    auto emit = [&](int gy, const int (&xu)[4], const int (&xm)[4], const int (&xd)[4], const int (&yu)[4],
                    const int (&ym)[4], const int (&yd)[4], const int (&zu)[4], const int (&zm)[4],
                    const int (&zd)[4]) {
        uint32_t packed = 0;
        float rv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int sxx = box_round(xu[i] + xm[i] + xd[i]);
            const int syy = box_round(yu[i] + ym[i] + yd[i]);
            const int sxy = box_round(zu[i] + zm[i] + zd[i]);
            const long long det = static_cast<long long>(sxx) * syy - static_cast<long long>(sxy) * sxy;
            const long long tr = static_cast<long long>(sxx) + syy;
            const double r = __dsub_rn(__ll2double_rn(det), __dmul_rn(p.k, __ll2double_rn(tr * tr)));
            const float rf = __double2float_rn(r);
            rv[i] = rf;
            const uint32_t m = static_cast<double>(rf) > p.threshold ? 255u : 0u;
            packed |= m << (8 * i);
        }
        const int row = gy - p.band.dst_row0;
        uint8_t* mp = mrow_base + static_cast<int64_t>(row) * p.mask_pitch + c;
        if (c + 3 < p.width) {
            *reinterpret_cast<uint32_t*>(mp) = packed;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (c + i < p.width) mp[i] = static_cast<uint8_t>(packed >> (8 * i));
        }
        if (kResp) {
            float* rp = reinterpret_cast<float*>(rrow_base + static_cast<int64_t>(row) * p.resp_pitch) + c;
            if (c + 3 < p.width) {
                *reinterpret_cast<float4*>(rp) = make_float4(rv[0], rv[1], rv[2], rv[3]);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (c + i < p.width) rp[i] = rv[i];
            }
        }
    };

    // smem row j <-> global y0-2+j.  Step j: Sobel terms of row j; Sobel row
    // j-1 (products, horizontal box sums) at j >= 2; output row j-2 at j >= 4.
    const int steps = (y1 - y0) + 4;
    auto step = [&](int j, int (&da)[6], int (&db)[6], int (&dc)[6], int (&sa)[6], int (&sb)[6], int (&sc)[6],
                    int (&xa)[4], int (&xb)[4], int (&xc)[4], int (&ya)[4], int (&yb)[4], int (&yc)[4],
                    int (&za)[4], int (&zb)[4], int (&zc)[4]) {
        int s[8];
        fetch8h(tile + j * kHarSW, off, s);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            dc[k] = s[k + 2] - s[k];
            sc[k] = s[k] + 2 * s[k + 1] + s[k + 2];
        }
        if (j < 2) return;
        int px[6], py[6], pxy[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int gx = da[k] + 2 * db[k] + dc[k];
            const int gy = sc[k] - sa[k];
            px[k] = gx * gx;
            py[k] = gy * gy;
            pxy[k] = gx * gy;
        }
        if (klo == 0) {
            px[0] = px[1];
            py[0] = py[1];
            pxy[0] = pxy[1];
        }
        int ex = px[1], ey = py[1], exy = pxy[1]; // last in-image column (static indices)
#pragma unroll
        for (int k = 2; k < 6; ++k)
            if (k - 1 <= khi) {
                ex = px[k];
                ey = py[k];
                exy = pxy[k];
            }
#pragma unroll
        for (int k = 1; k < 6; ++k)
            if (k - 1 > khi) {
                px[k] = ex;
                py[k] = ey;
                pxy[k] = exy;
            }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            xc[i] = px[i] + px[i + 1] + px[i + 2];
            yc[i] = py[i] + py[i + 1] + py[i + 2];
            zc[i] = pxy[i] + pxy[i + 1] + pxy[i + 2];
        }
        if (j < 4) return;
        const int gy = y0 - 4 + j;
        const bool t = gy == 0, b = gy == H - 1; // product rows clamp into the image
        emit(gy, t ? xb : xa, xb, b ? xb : xc, t ? yb : ya, yb, b ? yb : yc, t ? zb : za, zb, b ? zb : zc);
    };
    for (int j = 0; j < steps; j += 3) {
        step(j, dA, dB, dC, sA, sB, sC, xA, xB, xC, yA, yB, yC, zA, zB, zC);
        if (j + 1 < steps) step(j + 1, dB, dC, dA, sB, sC, sA, xB, xC, xA, yB, yC, yA, zB, zC, zA);
        if (j + 2 < steps) step(j + 2, dC, dA, dB, sC, sA, sB, xC, xA, xB, yC, yA, yB, zC, zA, zB);
    }
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
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, kHarSW, kHarSH)) return rc;
    HarrisParams p;
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
    const int frames = s.frames > 0 ? s.frames : 1;
    dim3 grid((s.width + kHarTW - 1) / kHarTW, (rows + kHarTH - 1) / kHarTH, frames);
    void* args[] = {&map, &p};
    void* fn = p.resp ? reinterpret_cast<void*>(&harris_kernel<true>) : reinterpret_cast<void*>(&harris_kernel<false>);
    cudaError_t e = cudaLaunchKernel(fn, grid, dim3(kHarThreads), args, 0, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "harris kernel launch");
    return check_launch(ctx, "harris kernel");
}
