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
/// SW must be a multiple of 16 and <= 1024; the tile base 128-byte aligned;
/// x_org MUST be a multiple of 16: a tiled TMA box whose inner start
/// coordinate is not 16-byte aligned faults with "illegal instruction" on
/// B200 (measured).
/// `sh` (<= SH) rows are loaded: the tensor map's box height (a tile of
/// sh - halo output rows, chosen per launch to fill whole waves).
template <int SW, int SH>
__device__ __forceinline__ void stage_tile_u8(uint8_t* tile, const CUtensorMap* map, uint64_t* bar, int x_org,
                                              int y_org, int frame, int width, const Band& band, int sh = SH) {
    static_assert(SW % 16 == 0 && SW <= 1024 && SH <= 256, "bad tile geometry");
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, SW * sh);
        tma_load_3d(tile, map, bar, x_org / 4, y_org - band.src_row0, frame);
    }
    mbar_wait(bar, 0);

    const bool left = x_org < 0;
    const bool right = x_org + SW > width;
    const bool top = y_org < 0;
    const bool bottom = y_org + sh > band.global_h;
    if (!(left | right | top | bottom)) return; // block-uniform

    // 1) replicate edge columns in rows that lie inside the image
    //    (warp per row, lane per column: no integer division on this path)
    const int nwarps = static_cast<int>(blockDim.x) >> 5, wid = static_cast<int>(threadIdx.x) >> 5;
    const int ln = static_cast<int>(threadIdx.x) & 31;
    if (left | right) {
        const int first = clampi(-x_org, 0, SW - 1);           // smem col of image col 0
        const int last = clampi(width - 1 - x_org, 0, SW - 1); // smem col of image col W-1
        for (int r = wid; r < sh; r += nwarps) {
            const int gy = y_org + r;
            if (gy < 0 || gy >= band.global_h) continue;
            uint8_t* row = tile + r * SW;
            const uint8_t vf = row[first], vl = row[last];
            // only the patched columns: [0, first) and (last, SW)
            for (int j = ln; j < first; j += 32) row[j] = vf;
            for (int j = last + 1 + ln; j < SW; j += 32) row[j] = vl;
        }
        __syncthreads();
    }
    // 2) replicate edge rows
    if (top | bottom) {
        for (int r = wid; r < sh; r += nwarps) {
            const int gy = y_org + r;
            if (gy >= 0 && gy < band.global_h) continue;
            const int src = clampi(gy, 0, band.global_h - 1) - y_org;
            const uint32_t* from = reinterpret_cast<const uint32_t*>(tile + src * SW);
            uint32_t* to = reinterpret_cast<uint32_t*>(tile + r * SW);
            for (int j = ln; j < SW / 4; j += 32) to[j] = from[j];
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
