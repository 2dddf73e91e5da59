/*
 * gvx_c.h — C facade of the graphvx-b200 graph API (in libgraphvx.so), for
 * FFI hosts (ctypes / cgo / JNI).  It drives the same public C++ entry
 * points a C++ user calls (verify, expand, optimize, run_plan, run_naive,
 * DeviceSession), so measurements through it are measurements of the API.
 *
 * Reference interfaces these wrap (ref = /root/reference/proj):
 *   gvxc_graph_*          Context / AppGraph / add_node / add_custom
 *                         (include/graphvx/graph.hpp:87-201, registry.hpp:48-64)
 *   gvxc_*_verify / plan  verify -> expand -> verify -> optimize
 *                         (verify.hpp:74, registry.hpp:70, optimize.hpp:109)
 *   gvxc_*_run_host       run_plan / run_naive (execute.hpp:60-65)
 *   gvxc_session_*        additive device-resident execution (device.hpp)
 * Status: 0 = ok, else gvx::ErrorCode + 1 (1..20) or 100+ for runtime
 * failures; gvxc_last_error() holds the message.
 */
#ifndef GVX_C_H_
#define GVX_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gvxc_graph_s* gvxc_graph;
typedef struct gvxc_session_s* gvxc_session;

const char* gvxc_last_error(void);
int gvxc_device_count(void);

/* ---- the five BASELINE configurations (config_graphs.hpp) ---------------- */
/* cfg 1..5; virtual_mid = 1 uses virtual intermediates (the fusible form). */
int gvxc_config_create(int cfg, int width, int height, int virtual_mid, gvxc_graph* out);
int gvxc_graph_destroy(gvxc_graph g);
/* Device program summary (naive = 1: per-node program, else the plan's). */
int gvxc_graph_describe(gvxc_graph g, int naive, char* buf, size_t cap);
/* PassStats of the optimized plan: {nodes_before, nodes_alive, removed,
 * transfers_naive, transfers_optimized, fused_groups, launches_before,
 * launches_after}. */
int gvxc_graph_pass_stats(gvxc_graph g, long long stats[8]);

/* Host-buffer execution through run_plan (naive = 0) / run_naive (1).
 * `in` = packed U8 input.  Outputs by config: cfg1/5 S16 plane, cfg2/3 U8
 * plane into `out`; cfg4 hist[256] + stats {mean, stddev}.  counters gets
 * {kernel_launches, pixels_read, pixels_written, transfers_executed}. */
int gvxc_graph_run_host(gvxc_graph g, int naive, const uint8_t* in, void* out, long long* hist, double* stats,
                        long long counters[4]);

/* ---- device-resident sessions ---------------------------------------------- */
int gvxc_session_create(gvxc_graph g, int naive, int frames, gvxc_session* out);
int gvxc_session_destroy(gvxc_session s);
/* slot 0 = the input image; slot k >= 1 = config output k-1. */
int gvxc_session_bind(gvxc_session s, int slot, void* dptr, int64_t pitch, int64_t frame_stride);
int gvxc_session_set_stream(gvxc_session s, void* cuda_stream);
/* Programmatic dependent launch of consecutive non-aliasing executions:
 * -1 own stream only (default), 0 off, 1 on (DeviceSession::set_overlap). */
int gvxc_session_set_overlap(gvxc_session s, int mode);
int gvxc_session_launch(gvxc_session s);
int gvxc_session_sync(gvxc_session s);
int gvxc_session_launches(gvxc_session s);
/* Host copies of one frame of slot 0 (upload) / output slot (download). */
int gvxc_session_upload_input(gvxc_session s, int frame, const uint8_t* in);
int gvxc_session_download(gvxc_session s, int slot, int frame, void* out, long long* hist, double* stats);

/* Device kernels launched so far by the library's device context. */
long long gvxc_launch_count(void);
/* The library's launch stream (cudaStream_t) for `device`'s context. */
void* gvxc_default_stream(void);

/* Reference-identical synthetic input (random_buffer, U8). */
int gvxc_random_u8(int width, int height, unsigned long long seed, uint8_t* out);

/* Zero-copy host runs: the graph's own page-locked input buffer (fill it and
 * pass it as `in` to gvxc_graph_run_host, or pass NULL), and the first image
 * output of the latest host run (valid until the next run). */
int gvxc_graph_input_ptr(gvxc_graph g, uint8_t** ptr, size_t* bytes);
int gvxc_graph_output_ptr(gvxc_graph g, const void** ptr, size_t* bytes);

/* Pipelined host runs (gvx::HostPipeline): up to `depth` frames in flight,
 * upload / kernels / download of consecutive frames overlapped.  submit
 * copies the frame; next returns the oldest frame's result in submission
 * order (same outputs / counters as gvxc_graph_run_host). */
typedef struct gvxc_pipeline_s* gvxc_pipeline;
int gvxc_pipeline_create(gvxc_graph g, int naive, int depth, gvxc_pipeline* out);
int gvxc_pipeline_destroy(gvxc_pipeline p);
int gvxc_pipeline_submit(gvxc_pipeline p, const uint8_t* in);
/* As gvxc_pipeline_submit without the staging copy: `in` must be page-locked
 * (gvxc_host_register) and stay unchanged until the frame's result is taken. */
int gvxc_pipeline_submit_pinned(gvxc_pipeline p, const uint8_t* in);
/* Page-lock / release caller memory (cudaHostRegister) for the pinned submit. */
int gvxc_host_register(void* ptr, size_t bytes);
int gvxc_host_unregister(void* ptr);
int gvxc_pipeline_pending(gvxc_pipeline p);
int gvxc_pipeline_next(gvxc_pipeline p, void* out, long long* hist, double* stats, long long counters[4]);
/* As gvxc_pipeline_next for image-output graphs, without the copy: *view
 * points at the result in page-locked staging until the next submit. */
int gvxc_pipeline_next_view(gvxc_pipeline p, const void** view, size_t* bytes, long long counters[4]);
/* A stream of n host frames through the pipeline in one call (image-output
 * graphs): keeps `depth` frames in flight and hands every result, in order,
 * to on_result (may be NULL) while it is still in page-locked staging;
 * counters = sums over the frames.  `pinned`: frames are page-locked
 * (gvxc_host_register) and DMAed without the staging copy. */
int gvxc_pipeline_stream(gvxc_pipeline p, const uint8_t* const* frames, int n, int pinned,
                         void (*on_result)(const void* view, size_t bytes, void* user), void* user,
                         long long counters[4]);

/* ---- row bands across GPUs (gvx::BandedSession / gvx::BandGroup) ---------
 * Slots as for sessions (0 = the input image, k >= 1 = config output k-1).
 * comm: a gvxb_comm (NCCL, one process per GPU) or NULL for world == 1;
 * device -1 = the library's device.  Rows are global image rows. */
typedef struct gvxc_band_s* gvxc_band;
typedef struct gvxc_group_s* gvxc_group;
int gvxc_band_create(gvxc_graph g, int rank, int world, void* comm, int device, int frames, gvxc_band* out);
int gvxc_band_destroy(gvxc_band b);
/* {rank, world, width, height, row0, row1, src_row0, src_row1, halo} */
int gvxc_band_layout(gvxc_band b, int32_t out[9]);
int gvxc_band_tensor(gvxc_band b, int slot, void** dptr, int64_t* pitch, int64_t* fstride, int32_t* first_row,
                     int32_t* rows);
int gvxc_band_upload(gvxc_band b, int slot, const void* host, size_t pitch, int first_row, int rows, int frame);
int gvxc_band_download(gvxc_band b, int slot, void* host, size_t pitch, int first_row, int rows, int frame);
int gvxc_band_set_stream(gvxc_band b, void* stream);
int gvxc_band_set_overlap(gvxc_band b, int mode);
/* Caller storage for a slot's band rows (as gvxc_band_tensor reports them). */
int gvxc_band_bind(gvxc_band b, int slot, void* dptr, int64_t pitch, int64_t fstride);
int gvxc_band_launch(gvxc_band b);
int gvxc_band_sync(gvxc_band b);
int gvxc_band_launches(gvxc_band b);
/* End to end from host memory: src = input slab rows [src_row0, src_row1),
 * dst = output rows [row0, row1) of `slot`; pieces pipelined (upload, kernel,
 * download on three streams); returns when dst is complete. */
int gvxc_band_run_host(gvxc_band b, const void* src, size_t src_pitch, int slot, void* dst, size_t dst_pitch,
                       int piece_rows);
int gvxc_band_describe(gvxc_band b, char* buf, size_t cap);
/* n bands of one image in this process, band i on devices[i] (entries may
 * repeat); halo rows move by strided peer copies.  gvxc_group_band returns a
 * borrowed handle (destroyed with the group). */
int gvxc_group_create(gvxc_graph g, int n, const int* devices, int frames, gvxc_group* out);
int gvxc_group_destroy(gvxc_group gr);
int gvxc_group_band(gvxc_group gr, int i, gvxc_band* out);
int gvxc_group_launch(gvxc_group gr);
int gvxc_group_sync(gvxc_group gr);

/* ---- graph description files (graph_io.hpp, ref:src/graph_io.cpp) -------- */
typedef struct gvxc_json_s* gvxc_json;
/* save_graph_json(load_graph_json(text)); *len = bytes needed (incl. NUL). */
int gvxc_json_roundtrip(const char* text, char* out, size_t cap, size_t* len);
/* load -> verify -> expand -> verify -> optimize. */
int gvxc_json_load(const char* text, gvxc_json* out);
int gvxc_json_destroy(gvxc_json g);
/* Runs with random_buffer(desc, seed + id) for every non-virtual source
 * image; writes the declared outputs serialised as [u32 kind][u32 n][bytes]
 * (configs/json_runner.hpp); *len = bytes needed; counters as in
 * gvxc_graph_run_host. */
int gvxc_json_run(gvxc_json g, int naive, unsigned long long seed, uint8_t* out, size_t cap, size_t* len,
                  long long counters[4]);
/* PassStats of the plan (same layout as gvxc_graph_pass_stats). */
int gvxc_json_pass_stats(gvxc_json g, long long st[8]);
/* Device benchmark of the graph through DeviceSession (plan or naive):
 * `frames` frames per execution (random_buffer inputs, seed + id), `iters`
 * timed executions.  out = {ms per execution, algorithmic HBM bytes per
 * execution (non-virtual source images read + produced images written),
 * kernel launches per execution, frames}. */
int gvxc_json_bench(gvxc_json g, int naive, int frames, int iters, unsigned long long seed, double out[4]);
/* Device program summary (naive = 1: per-node program, else the plan's). */
int gvxc_json_describe(gvxc_json g, int naive, char* buf, size_t cap);

#ifdef __cplusplus
}
#endif

#endif /* GVX_C_H_ */
