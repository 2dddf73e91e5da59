/*
 * gvxb.h — C-ABI of the graphvx-b200 device runtime (libgvx_cuda.so).
 *
 * This is the drop-in boundary between the unchanged C++ graph API
 * (include/graphvx/ headers, which keeps the reference's vxCreateGraph /
 * vxVerifyGraph / vxProcessGraph surface) and the hand-written sm_100a
 * kernels.  Plain C: POD structs, raw pointers, sizes and int status codes;
 * no C++ or torch types cross it.  Every function returns GVXB_OK (0) or a
 * status; gvxb_last_error() gives the thread's last message.
 *
 * Which reference interface each group replaces (the reference has no FFI:
 * these are the internal seams of its CPU engine, ref = /root/reference/proj):
 *   contexts, memory, copies     Engine::bind_inputs / buffer_of / the
 *                                Buffer store (ref:src/execute.cpp:300-359)
 *   gvxb_edge_*                  Engine::exec_local + exec_point for the
 *                                Gaussian3x3 -> Sobel3x3 -> Magnitude chain
 *                                (ref:src/execute.cpp:421-622,
 *                                 ref:src/registry.cpp:555-575,722-784)
 *   gvxb_harris                  exec_local/exec_point for the Harris chain
 *                                (Sobel, Multiply, Box3x3, user point nodes)
 *   gvxb_stencil_point           exec_local of a user-defined linear local
 *                                node fused with its point consumers
 *                                (ref:src/execute.cpp:504-622, optimize.cpp:393-441)
 *   gvxb_conv_stats              exec_local (Convolve) + exec_point
 *                                (ConvertDepth) + exec_histogram +
 *                                exec_reduce (ref:src/execute.cpp:624-727)
 *   gvxb_jit_*                   the per-node interpreter
 *                                (CompiledExpr::run, ref:src/expr.cpp:486-519)
 *                                replaced by CUDA C emitted from the
 *                                expression IR and compiled with NVRTC for
 *                                sm_100a (generic / run_naive path)
 *   gvxb_band_*                  no reference counterpart (row bands across
 *                                GPUs with halo rows; the reference splits
 *                                rows over <= 4 host threads,
 *                                ref:src/execute.cpp:392-419)
 */
#ifndef GVXB_H_
#define GVXB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GVXB_ABI_VERSION 1

/* ---- status codes --------------------------------------------------------
 * 1..20 mirror gvx::ErrorCode + 1 (error.hpp) so the host maps them 1:1. */
#define GVXB_OK 0
#define GVXB_ERR_SHAPE_MISMATCH 12 /* gvx::ErrorCode::ShapeMismatch + 1 */
#define GVXB_ERR_DIV_BY_ZERO 13    /* gvx::ErrorCode::DivByZero + 1 */
#define GVXB_ERR_UNSUPPORTED 17    /* gvx::ErrorCode::UnsupportedKind + 1 */
#define GVXB_ERR_CUDA 100
#define GVXB_ERR_NVRTC 101
#define GVXB_ERR_NO_DEVICE 102
#define GVXB_ERR_INVALID 103

/* device status word bits raised by kernels (read with gvxb_status_read) */
#define GVXB_STATUS_DIV_BY_ZERO 1u
#define GVXB_STATUS_INDEX_RANGE 2u

/* pixel formats: numeric values of gvx::ImageFormat */
#define GVXB_U8 0
#define GVXB_U16 1
#define GVXB_S16 2
#define GVXB_S32 3
#define GVXB_F32 4
#define GVXB_RGB 5
#define GVXB_UYVY 6

/* Device layout of a scalar / array element / matrix element: the
 * reference's tagged Value (ref:include/graphvx/value.hpp:14-40).
 * real != 0: bits holds an IEEE double; else bits is the int64. */
typedef struct gvxb_value {
    int64_t real;
    int64_t bits;
} gvxb_value;

typedef struct gvxb_ctx_s* gvxb_ctx;
typedef struct gvxb_module_s* gvxb_module;

/* A device image (or a stack of `frames` images `frame_stride` bytes apart).
 * Rows are `pitch` bytes apart; pitch is a multiple of 16 for TMA. */
typedef struct gvxb_image {
    void* data;
    int64_t pitch;
    int32_t width;
    int32_t height;
    int32_t format;
    int32_t frames;
    int64_t frame_stride;
} gvxb_image;

/* ---- runtime ------------------------------------------------------------ */
const char* gvxb_last_error(void);
int gvxb_abi_version(void);
int gvxb_device_count(int* count);
int gvxb_ctx_create(int device, gvxb_ctx* out);
int gvxb_ctx_destroy(gvxb_ctx ctx);
/* Launch on an external stream (e.g. a framework's); NULL = own stream. */
int gvxb_ctx_set_stream(gvxb_ctx ctx, void* cuda_stream);
/* Programmatic dependent launch of the hand-written kernels: a kernel whose
 * read / write ranges do not touch the previous kernel's (on this context's
 * stream, with nothing else enqueued in between) is launched so that it
 * starts while the previous one drains; a dependent one still starts early
 * but waits for it (griddepcontrol.wait) before touching memory.  mode
 * -1 (default) = only while the context launches on its own stream (then no
 * foreign work can sit between two of its kernels), 0 = off, 1 = on (the
 * caller guarantees that nothing else launches kernels on the stream). */
int gvxb_ctx_set_overlap(gvxb_ctx ctx, int mode);
void* gvxb_ctx_stream(gvxb_ctx ctx);
int gvxb_ctx_device(gvxb_ctx ctx);
int gvxb_ctx_sm_count(gvxb_ctx ctx);
int gvxb_sync(gvxb_ctx ctx);
/* Number of device kernels this context launched so far. */
int64_t gvxb_launch_count(gvxb_ctx ctx);
/* Kernels launched by every context of the process. */
int64_t gvxb_total_launch_count(void);

/* ---- memory and copies ---------------------------------------------------- */
int gvxb_alloc(gvxb_ctx ctx, size_t bytes, void** dptr);
int gvxb_free(gvxb_ctx ctx, void* dptr);
/* Debugging aid (compute-sanitizer stand-in): with GVX_GUARD_ALLOC=1 in the
 * environment every gvxb_alloc is framed by 4 KB of 0xA5 guard bytes that
 * gvxb_free checks.  Returns the number of allocations whose guards were
 * found overwritten (freed ones plus the still-live ones, checked now);
 * *live (may be null) = allocations still live.  0 without the mode. */
int64_t gvxb_guard_check(int* live);
int gvxb_host_alloc(size_t bytes, void** hptr); /* pinned */
int gvxb_host_free(void* hptr);
/* Page-lock existing host memory (cudaHostRegister) so copies DMA from/to it
 * directly; gvxb_host_is_pinned reports whether [ptr, ptr+bytes) is. */
int gvxb_host_register(void* hptr, size_t bytes);
int gvxb_host_unregister(void* hptr);
int gvxb_host_is_pinned(const void* hptr, int* pinned);
int gvxb_memset(gvxb_ctx ctx, void* dptr, int value, size_t bytes);
int gvxb_upload_2d(gvxb_ctx ctx, void* dst, size_t dpitch, const void* src, size_t spitch,
                   size_t row_bytes, size_t rows);
int gvxb_download_2d(gvxb_ctx ctx, void* dst, size_t dpitch, const void* src, size_t spitch,
                     size_t row_bytes, size_t rows);
int gvxb_copy_d2d(gvxb_ctx ctx, void* dst, const void* src, size_t bytes);

/* ---- timing (CUDA events on the context's stream) -------------------------- */
int gvxb_event_create(void** ev);
int gvxb_event_destroy(void* ev);
int gvxb_event_record(gvxb_ctx ctx, void* ev);
int gvxb_event_elapsed_ms(void* start, void* stop, float* ms);
int gvxb_event_sync(void* ev); /* host waits for the event */

/* ---- device status word / event counters ----------------------------------- */
int gvxb_status_reset(gvxb_ctx ctx);
/* Status word and read counter in one device->host read (one sync). */
int gvxb_status_counter_read(gvxb_ctx ctx, uint32_t* status, long long* counter);
/* Synchronises; returns the OR of GVXB_STATUS_* raised since the reset. */
int gvxb_status_read(gvxb_ctx ctx, uint32_t* status);
/* Device addresses of the status word and of the read counter (the
 * generated kernels receive them as parameters). */
int gvxb_status_ptr(gvxb_ctx ctx, uint32_t** dptr);
/* Device-side read counter used by generated kernels (reference event model). */
int gvxb_counter_ptr(gvxb_ctx ctx, unsigned long long** dptr);
int gvxb_counter_read(gvxb_ctx ctx, long long* reads);

/* ---- hand-written fused kernels -------------------------------------------
 * Row bands: a kernel computes output rows [row0, row1) of an image whose
 * global height is `global_h`; `src` holds global rows
 * [src_row0, src_row0 + src.height).  Clamp semantics use global rows, so a
 * band whose source carries the halo rows reproduces the single-GPU result.
 * For a whole image: row0 = 0, row1 = global_h = src.height, src_row0 = 0. */
typedef struct gvxb_band {
    int32_t row0, row1;
    int32_t global_h;
    int32_t src_row0;
    int32_t dst_row0; /* global row stored at dst row 0 */
} gvxb_band;

/* Gaussian3x3 (optional) -> Sobel3x3 -> {gx, gy, Magnitude}; U8 -> S16.
 * Null `data` in gx / gy / mag skips that output. */
typedef struct gvxb_edge_args {
    gvxb_image src;
    gvxb_image gx, gy, mag;
    int32_t with_gauss;
    gvxb_band band;
} gvxb_edge_args;
int gvxb_edge(gvxb_ctx ctx, const gvxb_edge_args* a);

/* Harris: Sobel -> Ixx/Iyy/Ixy (S32) -> Box3x3 -> response
 * F32((Sxx*Syy - Sxy^2) - k*(Sxx+Syy)^2) -> U8 mask (resp > threshold).
 * Optional debug outputs (null data = skip): response (F32). */
typedef struct gvxb_harris_args {
    gvxb_image src;
    gvxb_image mask;
    gvxb_image response;
    double k;
    double threshold;
    gvxb_band band;
} gvxb_harris_args;
int gvxb_harris(gvxb_ctx ctx, const gvxb_harris_args* a);

/* Linear integer stencil (odd ksize <= 7, Clamp) over U8 with an epilogue
 * chain.  s = sum(mask * window).  stage value b = sat(round_shift(s)) to
 * blur_format; then the point chain:
 *   mode 0: out = sat_U8(b)                             (blur only)
 *   mode 1: out = sat_U8(sat_S16(x + sat_S16(x - b)))   (unsharp: Add(in, Subtract(in, blur)) -> ConvertDepth)
 * round_shift: (s * num) / den with round-half-away and den = 2^shift or odd. */
typedef struct gvxb_stencil_args {
    gvxb_image src;
    gvxb_image dst;
    int32_t ksize;
    int32_t mask[49];
    int64_t div_num;  /* post-body factor = div_num / div_den (exact) */
    int64_t div_den;
    int32_t mode;
    gvxb_band band;
} gvxb_stencil_args;
int gvxb_stencil_point(gvxb_ctx ctx, const gvxb_stencil_args* a);

/* Convolve(kxk, scale) -> ConvertDepth(S16->U8, shift, policy) ->
 * {Histogram(bins, offset, range), sum, sum of squares} per frame, plus the
 * MeanStdDev finalize (IEEE double, no FMA) into mean[f] / stddev[f].
 * src.frames frames processed. */
typedef struct gvxb_conv_stats_args {
    gvxb_image src;
    gvxb_image converted;  /* optional: store the U8 image (null = virtual) */
    int32_t ksize;
    int32_t mask[49];
    int64_t scale;
    int32_t conv_format;   /* format of the convolve output (S16 / U8) */
    int32_t shift;
    int32_t wrap;
    int32_t bins;
    int64_t offset;
    int64_t range;
    gvxb_value* hist;      /* frames x bins integer counts (may be null) */
    int64_t* sum;          /* frames int64 scratch (required) */
    int64_t* sumsq;        /* frames int64 scratch (required) */
    gvxb_value* mean;      /* frames, F32-rounded real (may be null) */
    gvxb_value* stddev;    /* frames, F32-rounded real (may be null) */
    int64_t* work;         /* optional: frames x (bins + 1) int64, zero on entry (allocate zeroed
                              once; each call leaves it and sum / sumsq zero again): with it a
                              single frame is one launch (the kernel's last CTA publishes hist /
                              mean / stddev); without it, or for several frames, a scratch clear
                              and a finalize kernel bracket the convolution */
} gvxb_conv_stats_args;
int gvxb_conv_stats(gvxb_ctx ctx, const gvxb_conv_stats_args* a);

/* ---- generic path: NVRTC-compiled kernels from the expression IR ---------- */
int gvxb_jit_build(gvxb_ctx ctx, const char* source, const char* const* kernel_names, int n_kernels,
                   gvxb_module* out);
int gvxb_jit_free(gvxb_module m);
int gvxb_jit_launch(gvxb_ctx ctx, gvxb_module m, int kernel_index, const unsigned grid[3],
                    const unsigned block[3], size_t smem_bytes, void** args);
/* NVRTC log of the last failed build on this thread. */
const char* gvxb_jit_log(void);

/* ---- multi-GPU row bands -------------------------------------------------
 * No reference counterpart: the reference splits rows over <= 4 host
 * threads (ref:src/execute.cpp:392-419).  Band g of G owns global output
 * rows [row0, row1); a stencil group of radius R reads source rows
 * [row0 - R, row1 + R) clipped to the image (its "slab"); the R rows on each
 * side that it does not own come from its neighbours once per group
 * execution. */

/* Rows of band `rank` of `world` for an image of height h (balanced split). */
int gvxb_band_rows(int32_t h, int32_t world, int32_t rank, int32_t* row0, int32_t* row1);

/* One band's rows, overlap split and exchange schedule.  Side 0 is the
 * upper neighbour (rank - 1), side 1 the lower (rank + 1); peer[s] = -1 when
 * absent.  Interior rows read owned source rows only (computed while the
 * halo rows are in flight); the edge rows read halo rows.  For world > 1
 * every band must be at least `halo` rows tall (neighbours supply the whole
 * halo). */
typedef struct gvxb_band_plan {
    int32_t height, world, rank, halo;
    int32_t row0, row1;                   /* owned output rows */
    int32_t src_row0, src_row1;           /* slab rows (owned + halo, clipped) */
    int32_t interior_row0, interior_row1; /* empty when interior_row0 == interior_row1 */
    int32_t n_edges;
    int32_t edge_row0[2], edge_row1[2];
    int32_t peer[2];
    int32_t send_row0[2], send_rows[2];   /* my owned rows sent to peer[s] */
    int32_t recv_row0[2], recv_rows[2];   /* halo rows received from peer[s] */
} gvxb_band_plan;
int gvxb_band_plan_make(int32_t height, int32_t world, int32_t rank, int32_t halo, gvxb_band_plan* out);

/* Enable peer access from ctx's device to `peer_device` (NVLink P2P). */
int gvxb_enable_peer(gvxb_ctx ctx, int peer_device);
/* Copy `rows` rows of `row_bytes` between (possibly different) devices as
 * one strided DMA (cudaMemcpy3DPeerAsync) on ctx's stream. */
int gvxb_copy_peer_rows(gvxb_ctx ctx, void* dst, size_t dpitch, int dst_device, const void* src,
                        size_t spitch, int src_device, size_t row_bytes, size_t rows);
/* ctx's stream waits for `ev` (recorded on any stream / device). */
int gvxb_stream_wait_event(gvxb_ctx ctx, void* ev);

/* NCCL communicator for the halo exchange between processes (one rank per
 * GPU).  NCCL is loaded at first use (dlopen "libnccl.so.2");
 * gvxb_comm_available() reports whether it could be. */
#define GVXB_COMM_ID_BYTES 128
typedef struct gvxb_comm_s* gvxb_comm;
int gvxb_comm_available(void);
int gvxb_comm_unique_id(uint8_t id[GVXB_COMM_ID_BYTES]);
int gvxb_comm_create(int device, int rank, int world, const uint8_t id[GVXB_COMM_ID_BYTES], gvxb_comm* out);
int gvxb_comm_destroy(gvxb_comm c);
/* Posts the halo exchange of `plan` for every frame of `slab` (an image
 * holding global rows [plan->src_row0, plan->src_row1)) on the
 * communicator's stream, ordered after ctx's enqueued work; returns at
 * once.  gvxb_halo_wait makes ctx's stream wait for it (sends included). */
int gvxb_halo_start(gvxb_ctx ctx, gvxb_comm c, const gvxb_band_plan* plan, const gvxb_image* slab);
int gvxb_halo_wait(gvxb_ctx ctx, gvxb_comm c);
/* Host-value max over ranks (blocking); barrier = an all-reduce. */
int gvxb_comm_allreduce_max(gvxb_comm c, double* value);
int gvxb_comm_barrier(gvxb_comm c);

#ifdef __cplusplus
}
#endif

#endif /* GVXB_H_ */
