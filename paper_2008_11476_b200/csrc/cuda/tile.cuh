// TMA tile staging with Clamp-border patching, shared by the fused stencil
// kernels.  One elected thread issues cp.async.bulk.tensor box loads on an
// mbarrier; all threads then replicate edge columns / rows for tiles that
// touch the image border, so the interior compute never branches on
// borders (the reference clamps every window read, ref:src/execute.cpp:242-245).
#pragma once

#include "common.cuh"

namespace gvxd {

struct Band {
    int row0, row1;  // output rows (global)
    int global_h;
    int src_row0;    // global row of source buffer row 0
    int dst_row0;    // global row of destination buffer row 0
};

/// smem tile: image columns [x_org, x_org + SW), global rows [y_org, y_org + SH),
/// one TMA box (the map views the plane as u32, see make_u8_tensor_map).
/// SW must be a multiple of 16 and <= 1024; x_org a multiple of 4; the
/// tile base 128-byte aligned.
template <int SW, int SH>
__device__ __forceinline__ void stage_tile_u8(uint8_t* tile, const CUtensorMap* map, uint64_t* bar, int x_org,
                                              int y_org, int frame, int width, const Band& band) {
    static_assert(SW % 16 == 0 && SW <= 1024 && SH <= 256, "bad tile geometry");
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, SW * SH);
        tma_load_3d(tile, map, bar, x_org / 4, y_org - band.src_row0, frame);
    }
    mbar_wait(bar, 0);

    const bool left = x_org < 0;
    const bool right = x_org + SW > width;
    const bool top = y_org < 0;
    const bool bottom = y_org + SH > band.global_h;
    if (!(left | right | top | bottom)) return; // block-uniform

    // 1) replicate edge columns in rows that lie inside the image
    if (left | right) {
        const int first = clampi(-x_org, 0, SW - 1);           // smem col of image col 0
        const int last = clampi(width - 1 - x_org, 0, SW - 1); // smem col of image col W-1
        for (int i = threadIdx.x; i < SH * SW; i += blockDim.x) {
            const int r = i / SW, j = i - r * SW;
            const int gy = y_org + r;
            if (gy < 0 || gy >= band.global_h) continue;
            if (j < first) tile[r * SW + j] = tile[r * SW + first];
            else if (j > last) tile[r * SW + j] = tile[r * SW + last];
        }
        __syncthreads();
    }
    // 2) replicate edge rows
    if (top | bottom) {
        for (int i = threadIdx.x; i < SH * SW; i += blockDim.x) {
            const int r = i / SW, j = i - r * SW;
            const int gy = y_org + r;
            if (gy >= 0 && gy < band.global_h) continue;
            const int src = clampi(gy, 0, band.global_h - 1) - y_org;
            tile[r * SW + j] = tile[src * SW + j];
        }
        __syncthreads();
    }
}

/// Pixel bytes of a 32-bit word at smem byte offset `off` (4-byte aligned).
__device__ __forceinline__ uint32_t lds32(const uint8_t* tile, int off) {
    return *reinterpret_cast<const uint32_t*>(tile + off);
}

__device__ __forceinline__ int byte_of(uint32_t w, int k) { return (w >> (8 * k)) & 0xFF; }

} // namespace gvxd
