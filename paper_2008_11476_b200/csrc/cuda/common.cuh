// Shared pieces of the sm_100a kernels: context layout, exact integer
// rounding helpers matching the reference's cast semantics, TMA/mbarrier
// wrappers, and the tile loader that reproduces Clamp borders in shared
// memory.
#pragma once

#include "gvxb.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

/// Device byte range [lo, hi) a kernel reads or writes.
struct gvxb_range {
    uintptr_t lo = 0, hi = 0;
};

constexpr int kTrackedRanges = 32; // read / write ranges of the overlap window (see gvxb_ctx_s)

struct gvxb_ctx_s {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    unsigned* status = nullptr;            // GVXB_STATUS_* bits
    unsigned long long* counter = nullptr; // pixel-read events of generated kernels
    int64_t launches = 0;
    // Programmatic dependent launch between hand-written kernels
    // (gvxb_ctx_set_overlap).  The window holds the ranges read / written by
    // every kernel that may still be running: the kernels launched since
    // the last fully stream-ordered launch, all mutually independent (a grid
    // launched programmatically may finish before its predecessor, so a
    // later launch must be independent of the whole window to overlap).
    // Valid only while nothing else was enqueued after the last of them.  A
    // launch that depends on the window may still overlap it when the window
    // is a single kernel: its griddepcontrol.wait (pdl_wait) covers it.
    int overlap = -1; // -1 auto (own stream only), 0 off, 1 on
    bool prev_kernel = false; // the window is valid
    gvxb_range prev_r[kTrackedRanges], prev_w[kTrackedRanges];
    int prev_nr = 0, prev_nw = 0;
    int prev_launches = 0; // kernels in the window
};

namespace gvxb_impl {
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int check_launch(gvxb_ctx ctx, const char* what);

/// Bytes [p, p + n) as a tracked range; empty for a null pointer.
inline gvxb_range bytes_range(const void* p, size_t n) {
    gvxb_range r;
    if (!p || !n) return r;
    r.lo = reinterpret_cast<uintptr_t>(p);
    r.hi = r.lo + n;
    return r;
}

/// Bytes of buffer rows [first, first + n) of a single-frame image (all of
/// it for several frames); empty for a null image.  Band launches use it so
/// kernels on disjoint rows of one buffer count as independent.
inline gvxb_range rows_range(const gvxb_image& im, int first, int n) {
    gvxb_range r;
    if (!im.data || im.height <= 0 || n <= 0) return r;
    if (im.frames > 1) {
        const int64_t span = im.frame_stride * (im.frames - 1) + im.pitch * im.height;
        r.lo = reinterpret_cast<uintptr_t>(im.data);
        r.hi = r.lo + static_cast<uintptr_t>(span);
        return r;
    }
    first = first < 0 ? 0 : first;
    const int last = first + n > im.height ? im.height : first + n;
    if (last <= first) return r;
    r.lo = reinterpret_cast<uintptr_t>(im.data) + static_cast<uintptr_t>(static_cast<int64_t>(first) * im.pitch);
    r.hi = reinterpret_cast<uintptr_t>(im.data) + static_cast<uintptr_t>(static_cast<int64_t>(last) * im.pitch);
    return r;
}

/// Bytes an image (all its frames) spans; empty for a null image.
inline gvxb_range image_range(const gvxb_image& im) {
    gvxb_range r;
    if (!im.data || im.height <= 0) return r;
    const int64_t frames = im.frames > 1 ? im.frames : 1;
    const int64_t span = (frames > 1 ? im.frame_stride * (frames - 1) : 0) + im.pitch * im.height;
    r.lo = reinterpret_cast<uintptr_t>(im.data);
    r.hi = r.lo + static_cast<uintptr_t>(span);
    return r;
}

/// Whether a kernel reading `r` and writing `w` may overlap the previous
/// kernel on ctx's stream: no read-after-write, write-after-read or
/// write-after-write through any of the ranges.  Returns the value of the
/// kernel's `pdl_wait` parameter: 1 = must wait for the previous grid.
int pdl_must_wait(gvxb_ctx ctx, const gvxb_range* r, int nr, const gvxb_range* w, int nw);
/// Whether a launch_tracked of these ranges will overlap the previous
/// kernel on the stream (programmatic dependent launch without a wait):
/// overlapped launches hide a grid's tail behind its successor's head, so
/// the row-ring kernels pick taller bands for them.
bool launch_overlaps(gvxb_ctx ctx, const gvxb_range* r, int nr, const gvxb_range* w, int nw);

/// Launches `fn` on ctx's stream, as a programmatic dependent launch when
/// the context allows it and the overlap window permits (runtime.cu), and
/// records this kernel's ranges in the window.
int launch_tracked(gvxb_ctx ctx, const void* fn, dim3 grid, dim3 block, void** args, size_t smem,
                   const gvxb_range* r, int nr, const gvxb_range* w, int nw, const char* what);

/// Any other stream operation (copies, memsets, generated kernels).
inline void untracked_op(gvxb_ctx ctx) { ctx->prev_kernel = false; }
} // namespace gvxb_impl

namespace gvxd {
/// Kernel prologue for programmatic dependent launch: when this grid
/// depends on the previous one (pdl_wait), wait for it, then let the next
/// grid on the stream be scheduled as this one's CTAs retire.  Both
/// are no-ops for a kernel launched without the PDL attribute.
__device__ __forceinline__ void pdl_prologue(int pdl_wait) {
    // a waiting grid releases its dependents only after its wait: the next
    // launch's overlap window then no longer holds the grid waited for
    if (pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
} // namespace gvxd

namespace gvxd {

__host__ __device__ __forceinline__ int clampi(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

/// round-half-away-from-zero of s / d for d > 0 (llround semantics of the
/// reference's `cast_value(Saturate, s * (1.0 / d))` when that product is
/// exact enough; callers prove that per use).
__device__ __forceinline__ int round_div_away(int s, int d) {
    int a = s < 0 ? -s : s;
    int q = (2 * a + d) / (2 * d);
    return s < 0 ? -q : q;
}

__device__ __forceinline__ int sat_s16(int v) { return clampi(v, -32768, 32767); }
__device__ __forceinline__ int sat_u8(int v) { return clampi(v, 0, 255); }

/// round(sqrt(n)) with half away from zero, exact for 0 <= n < 2^24:
/// fp32 estimate then integer correction (k = largest integer with
/// k*k - k < n).  Matches llround(sqrt((double)n)) of the reference
/// (Magnitude, ref:src/registry.cpp:567-570).
__device__ __forceinline__ int round_sqrt_exact(int n) {
    float s = sqrtf(__int2float_rn(n));
    int k = __float2int_rd(s + 0.4995f);
    k += (n > k * k + k) ? 1 : 0;
    return k;
}

// ---- mbarrier + TMA (cp.async.bulk.tensor) --------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

/// Orders this thread's generic-proxy shared-memory writes before later
/// async-proxy (TMA) writes of the same bytes.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

} // namespace gvxd

namespace gvxb_impl {

/// Encodes a 3D (x, y, frame) U8 tensor map for a gvxb_image with the given
/// box; OOB elements are zero-filled (kernels patch Clamp borders after).
int make_u8_tensor_map(CUtensorMap* map, const gvxb_image& img, int box_w, int box_h);

/// Shared-memory tile of U8 source pixels covering image columns
/// [x_org, x_org + tw) and rows [y_org, y_org + th) of a frame, loaded by TMA
/// and patched so out-of-image positions hold the clamped (replicated)
/// pixel: exactly the reference's Clamp window reads
/// (NodeEnv::window, ref:src/execute.cpp:233-248).
struct TileGeom {
    int x_org, y_org; // image coordinates of smem (0, 0)
    int tw, th;       // tile extent in smem (tw multiple of 16)
};

} // namespace gvxb_impl

namespace gvxb_impl {

/// Rows per tile for a tiled stencil launch: tiles = strips * ceil(rows / th)
/// run in waves of `slots` resident CTAs and each tile also pays `halo`
/// extra rows, so pick th <= th_max minimising waves * (th + halo).
inline int balanced_tile_rows(long long strips, int rows, long long slots, int th_max, int halo, int th_min = 8) {
    if (slots < 1) slots = 1;
    int best = th_max;
    long long best_cost = -1;
    for (int th = th_max; th >= th_min; --th) {
        const long long tiles = strips * ((rows + th - 1) / th);
        const long long waves = (tiles + slots - 1) / slots;
        const long long cost = waves * (th + halo);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = th;
        }
        if (th >= rows) continue;
    }
    return best;
}

} // namespace gvxb_impl
