// K1 — fused Gaussian3x3 -> Sobel3x3 -> Magnitude (U8 -> S16), one pass.
//
// Reference semantics reproduced bit-exactly:
//   gaussian3x3  sat_U8(llround(sum(mask*win) * (1/16)))  == (s + 8) >> 4
//                (ref:src/registry.cpp:722-746; s in [0, 4080] -> exact)
//   sobel_x/y    sat_S16(sum(mask*win)), |v| <= 1020
//                (ref:src/registry.cpp:748-784)
//   magnitude    sat_S16(llround(sqrt((double)(gx*gx + gy*gy))))
//                (ref:src/registry.cpp:555-575) via gvxd::round_sqrt_exact
//   Clamp of the *intermediate*: the Gaussian at an out-of-image position is
//   the Gaussian of the clamped position (run_naive materialises it and the
//   Sobel window clamps into it, ref:src/execute.cpp:242-245).
//
// Layout: CTA = 128 threads, output tile 512 x 32; each thread owns 4
// adjacent columns and streams down the rows keeping the horizontal sums,
// the Gaussian rows and the Sobel windows in registers (a 3-row ring), so
// every input byte is read from HBM once (plus a 4-row halo) and every output
// written once: 1 B in + 2 B out per output (3 B/px algorithmic traffic).
#include "tile.cuh"

namespace gvxd {

constexpr int kEdgeThreads = 128;
constexpr int kEdgeTW = 4 * kEdgeThreads; // 512 output columns per CTA
constexpr int kEdgeTH = 32;               // output rows per CTA
constexpr int kEdgeSW = kEdgeTW + 64;     // smem columns [x0 - 32, x0 + 544)
constexpr int kEdgeSH = kEdgeTH + 4;      // smem rows    [y0 - 2, y0 + 34)
constexpr int kEdgeBox = 192;

struct OutPlane {
    int16_t* data;
    int64_t pitch;        // bytes
    int64_t frame_stride; // bytes
};

struct EdgeParams {
    int width;
    Band band;
    OutPlane gx, gy, mag;
};

__device__ __forceinline__ void store4(const OutPlane& o, int frame, int row, int c, int width, int v0, int v1,
                                       int v2, int v3) {
    char* base = reinterpret_cast<char*>(o.data) + frame * o.frame_stride + static_cast<int64_t>(row) * o.pitch;
    int16_t* p = reinterpret_cast<int16_t*>(base) + c;
    if (c + 3 < width) {
        uint2 w;
        w.x = (static_cast<uint32_t>(v0) & 0xFFFFu) | (static_cast<uint32_t>(v1) << 16);
        w.y = (static_cast<uint32_t>(v2) & 0xFFFFu) | (static_cast<uint32_t>(v3) << 16);
        *reinterpret_cast<uint2*>(p) = w;
    } else {
        const int v[4] = {v0, v1, v2, v3};
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (c + i < width) p[i] = static_cast<int16_t>(v[i]);
    }
}

/// 8 source bytes for columns c-2 .. c+5 from three aligned words.
__device__ __forceinline__ void fetch8(const uint8_t* row, int off, int (&a)[8]) {
    const uint32_t wl = lds32(row, off - 4), wc = lds32(row, off), wr = lds32(row, off + 4);
    a[0] = byte_of(wl, 2);
    a[1] = byte_of(wl, 3);
#pragma unroll
    for (int k = 0; k < 4; ++k) a[2 + k] = byte_of(wc, k);
    a[6] = byte_of(wr, 0);
    a[7] = byte_of(wr, 1);
}

template <bool kGauss, bool kGx, bool kGy, bool kMag>
__global__ void __launch_bounds__(kEdgeThreads) edge_kernel(const __grid_constant__ CUtensorMap map, EdgeParams p) {
    __shared__ alignas(128) uint8_t tile[kEdgeSH * kEdgeSW];
    __shared__ uint64_t bar;

    const int x0 = blockIdx.x * kEdgeTW;
    const int y0 = p.band.row0 + blockIdx.y * kEdgeTH;
    const int y1 = min(y0 + kEdgeTH, p.band.row1);
    const int frame = blockIdx.z;
    const int H = p.band.global_h;

    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    stage_tile_u8<kEdgeSW, kEdgeSH>(tile, &map, &bar, x0 - 32, y0 - 2, frame, p.width, p.band);

    const int c = x0 + 4 * static_cast<int>(threadIdx.x);
    if (c >= p.width) return;
    const int off = 4 * static_cast<int>(threadIdx.x) + 32; // smem column of c
    // horizontal clamp of the Gaussian intermediate: slot k (column c+k,
    // k = -1..4) reads the column clamped into the image
    const int klo = c == 0 ? 0 : -1;
    const int khi = min(4, p.width - 1 - c);

    int hA[6], hB[6], hC[6]; // horizontal Gaussian sums, 3-row ring
    int gA[6], gB[6], gC[6]; // Gaussian (or source) rows, columns c-1 .. c+4

    auto emit = [&](int gy, const int (&u)[6], const int (&m)[6], const int (&d)[6]) {
        // u = row gy-1, m = row gy, d = row gy+1 (after vertical clamping)
        int vx[4], vy[4], vm[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            vx[i] = (u[i + 2] - u[i]) + 2 * (m[i + 2] - m[i]) + (d[i + 2] - d[i]);
            vy[i] = (d[i] + 2 * d[i + 1] + d[i + 2]) - (u[i] + 2 * u[i + 1] + u[i + 2]);
            if (kMag) vm[i] = round_sqrt_exact(vx[i] * vx[i] + vy[i] * vy[i]);
        }
        const int row = gy - p.band.dst_row0;
        if (kGx) store4(p.gx, frame, row, c, p.width, vx[0], vx[1], vx[2], vx[3]);
        if (kGy) store4(p.gy, frame, row, c, p.width, vy[0], vy[1], vy[2], vy[3]);
        if (kMag) store4(p.mag, frame, row, c, p.width, vm[0], vm[1], vm[2], vm[3]);
    };

    if constexpr (kGauss) {
        // smem row j <-> global row y0-2+j; g(j-1) ready at step j >= 2;
        // output row y0-4+j ready at step j >= 4.
        const int steps = (y1 - y0) + 4;
        auto step = [&](int j, int (&a)[6], int (&b)[6], int (&cc)[6], int (&ga)[6], int (&gb)[6],
                        int (&gc)[6]) {
            int s[8];
            fetch8(tile + j * kEdgeSW, off, s);
#pragma unroll
            for (int k = 0; k < 6; ++k) cc[k] = s[k] + 2 * s[k + 1] + s[k + 2];
            if (klo == 0) cc[0] = cc[1];
            int edge = cc[1]; // value of the last in-image column (static indices only)
#pragma unroll
            for (int k = 2; k < 6; ++k)
                if (k - 1 <= khi) edge = cc[k];
#pragma unroll
            for (int k = 1; k < 6; ++k)
                if (k - 1 > khi) cc[k] = edge;
            if (j < 2) return;
#pragma unroll
            for (int k = 0; k < 6; ++k) gc[k] = (a[k] + 2 * b[k] + cc[k] + 8) >> 4;
            if (j < 4) return;
            const int gy = y0 - 4 + j;
            // vertical clamp of the intermediate: g(-1) := g(0), g(H) := g(H-1)
            emit(gy, gy == 0 ? gb : ga, gb, gy == H - 1 ? gb : gc);
        };
        for (int j = 0; j < steps; j += 3) {
            step(j, hA, hB, hC, gA, gB, gC);
            if (j + 1 < steps) step(j + 1, hB, hC, hA, gB, gC, gA);
            if (j + 2 < steps) step(j + 2, hC, hA, hB, gC, gA, gB);
        }
    } else {
        // Sobel straight on the source: g := input row (Clamp already in smem).
        // smem row j <-> global row y0-2+j; output row y0-3+j at step j >= 3.
        const int steps = (y1 - y0) + 3;
        auto step = [&](int j, int (&ga)[6], int (&gb)[6], int (&gc)[6]) {
            int s[8];
            fetch8(tile + j * kEdgeSW, off, s);
#pragma unroll
            for (int k = 0; k < 6; ++k) gc[k] = s[k + 1];
            if (j < 3) return;
            emit(y0 - 3 + j, ga, gb, gc);
        };
        (void)hA;
        (void)hB;
        (void)hC;
        for (int j = 1; j < steps; j += 3) {
            step(j, gA, gB, gC);
            if (j + 1 < steps) step(j + 1, gB, gC, gA);
            if (j + 2 < steps) step(j + 2, gC, gA, gB);
        }
    }
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
using EdgeFn = void (*)(const CUtensorMap, EdgeParams);

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

extern "C" int gvxb_edge(gvxb_ctx ctx, const gvxb_edge_args* a) {
    using namespace gvxb_impl;
    const gvxb_image& s = a->src;
    if (s.format != GVXB_U8) return fail(GVXB_ERR_INVALID, "edge: source must be U8");
    const bool ox = a->gx.data, oy = a->gy.data, om = a->mag.data;
    void* fn = a->with_gauss ? pick_edge<true>(ox, oy, om) : pick_edge<false>(ox, oy, om);
    if (!fn) return GVXB_OK; // nothing requested
    const int rows = a->band.row1 - a->band.row0;
    if (rows <= 0 || s.width <= 0) return GVXB_OK;
    CUtensorMap map;
    if (int rc = make_u8_tensor_map(&map, s, kEdgeSW, kEdgeSH)) return rc;
    EdgeParams p;
    p.width = s.width;
    p.band = Band{a->band.row0, a->band.row1, a->band.global_h, a->band.src_row0, a->band.dst_row0};
    p.gx = plane(a->gx);
    p.gy = plane(a->gy);
    p.mag = plane(a->mag);
    const int frames = s.frames > 0 ? s.frames : 1;
    dim3 grid((s.width + kEdgeTW - 1) / kEdgeTW, (rows + kEdgeTH - 1) / kEdgeTH, frames);
    void* args[] = {&map, &p};
    cudaError_t e = cudaLaunchKernel(fn, grid, dim3(kEdgeThreads), args, 0, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "edge kernel launch");
    return check_launch(ctx, "edge kernel");
}
