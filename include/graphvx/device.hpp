// graphvx-b200 — additive device-resident execution API (not in the
// reference).  run_plan / run_naive keep the reference's host-Buffer
// contract; DeviceSession launches the same lowered program on device
// buffers the caller owns (frame batches, benchmarks, multi-GPU bands) with
// no host copies on the critical path.
#pragma once

#include "graphvx/execute.hpp"

#include <memory>
#include <string>
#include <vector>

namespace gvx {

/// Caller-owned device storage for one non-virtual object.  Images: `pitch`
/// bytes per row (multiple of 16), frames `frame_stride` bytes apart.
/// Scalars / arrays: device Value slots (gvxb_value, 16 bytes each), frames
/// `frame_stride` bytes apart.
struct DeviceTensor {
    void* data = nullptr;
    std::int64_t pitch = 0;
    std::int64_t frame_stride = 0;
};

class DeviceSession {
public:
    /// Lowered optimized plan (fused device groups), `frames` per launch.
    explicit DeviceSession(const OptimizedPlan& plan, int frames = 1);
    /// Unfused program: one device kernel set per node (run_naive).
    explicit DeviceSession(const VerifiedGraph& g, int frames = 1);
    ~DeviceSession();
    DeviceSession(const DeviceSession&) = delete;
    DeviceSession& operator=(const DeviceSession&) = delete;

    /// Use caller memory for a non-virtual object (otherwise the session
    /// allocates it).
    void bind(ObjectId id, DeviceTensor t);
    /// Device storage the session uses for `id` (allocating if needed).
    DeviceTensor tensor(ObjectId id);

    /// Launch stream (a cudaStream_t); nullptr = the runtime's own stream.
    void set_stream(void* cuda_stream);
    /// Programmatic dependent launch between consecutive executions whose
    /// bound buffers do not alias (gvxb_ctx_set_overlap): -1 (default) only
    /// on the session's own stream, 0 off, 1 on (the caller guarantees no
    /// other kernels are launched on the stream set with set_stream).
    void set_overlap(int mode);
    /// Enqueue one execution of the program over all frames (asynchronous).
    void launch();
    /// Wait, then raise the reference's errors (DivByZero, ShapeMismatch)
    /// recorded by the kernels.
    void synchronize();

    void upload(ObjectId id, const Buffer& b, int frame = 0);
    Buffer download(ObjectId id, int frame = 0);

    int frames() const;
    int launches_per_run() const;
    std::string describe() const;

    struct Impl;

private:
    std::unique_ptr<Impl> impl_;
};

/// Pipelined host execution (additive): run_plan / run_naive semantics on
/// a stream of frames held in host Buffers, with up to `depth` frames in
/// flight.  Each slot owns device storage, a stream and page-locked
/// staging, so the upload of frame k+1, the kernels of frame k and the
/// download of frame k-1 overlap (two copy engines + the SMs).  Reports
/// come back in submission order and equal run_plan's / run_naive's.
class HostPipeline {
public:
    explicit HostPipeline(const OptimizedPlan& plan, int depth = 3);
    explicit HostPipeline(const VerifiedGraph& g, int depth = 3);
    ~HostPipeline();
    HostPipeline(const HostPipeline&) = delete;
    HostPipeline& operator=(const HostPipeline&) = delete;
    /// Copies the frame's inputs and enqueues it; when all slots are busy,
    /// first completes the oldest frame (its report waits for next()).
    void submit(const InputMap& inputs);
    /// FFI form: one image input from raw host memory (other inputs take
    /// the graph's bound values).
    void submit(ObjectId image_input, const void* data, std::size_t bytes);
    /// As the FFI submit, without the staging copy: `data` must be
    /// page-locked (gvxb_host_alloc / gvxb_host_register; ErrorCode::BadFormat
    /// otherwise) and is DMAed to the device directly, so the caller must
    /// leave it unchanged until this frame's result has been taken by
    /// next() / next_into() / next_view().
    void submit_pinned(ObjectId image_input, const void* data, std::size_t bytes);
    /// Report of the oldest submitted frame not yet returned (blocks).
    ExecutionReport next();
    /// As next(), but image output `image_output` is copied straight to
    /// `dst` (`bytes`, packed rows) and left out of the report.
    ExecutionReport next_into(ObjectId image_output, void* dst, std::size_t bytes);
    /// As next(), but image output `image_output` stays in the pipeline's
    /// page-locked staging: `*view` points at its packed rows, valid until
    /// the next submit().
    ExecutionReport next_view(ObjectId image_output, const void** view);
    /// Frames submitted and not yet returned by next().
    int pending() const;
    struct Impl;

private:
    std::unique_ptr<Impl> impl_;
};

/// Row-band geometry of one band (global rows; see gvxb_band_plan).
struct BandLayout {
    int rank = 0, world = 1;
    int width = 0, height = 0; ///< the whole image
    int row0 = 0, row1 = 0;    ///< owned output rows
    int src_row0 = 0, src_row1 = 0; ///< rows of the input slab (owned + halo)
    int halo = 0;              ///< total stencil radius of the program's input
};

class BandGroup;

/// Row-band execution of an optimized plan (additive; no reference
/// counterpart — the reference splits rows over <= 4 host threads,
/// ref:src/execute.cpp:392-419).  Band `rank` of `world` computes output
/// rows [row0, row1) of every image of the plan's device program.  Before
/// each fused stencil group, the halo rows of the group's input that the
/// band does not own come from its neighbours: over NCCL (`comm`, a
/// gvxb_comm, one process per GPU) or by peer copies inside a BandGroup;
/// Clamp borders use global rows, so the union of the bands equals the
/// single-image result bit for bit.  The exchange overlaps the interior rows,
/// which read owned rows only.  Programs must consist of hand-written
/// stencil groups over images of one size (Error(UnsupportedKind) otherwise).
namespace detail {
struct BandAccess;
}

class BandedSession {
public:
    BandedSession(const OptimizedPlan& plan, int rank, int world, void* comm = nullptr, int device = -1,
                  int frames = 1);
    ~BandedSession();
    BandedSession(const BandedSession&) = delete;
    BandedSession& operator=(const BandedSession&) = delete;

    BandLayout layout() const;
    /// Band storage of image `id`: its pointer addresses global row `first_row`
    /// (the slab's first row: src_row0 for an input, row0 for an output).
    DeviceTensor tensor(ObjectId id, int* first_row = nullptr, int* rows = nullptr);
    void set_stream(void* cuda_stream);
    /// As DeviceSession::set_overlap.
    void set_overlap(int mode);
    /// Use caller memory for image `id`'s band storage (same rows as
    /// tensor(id) reports; pitch a multiple of 16 and >= the row bytes),
    /// e.g. to alternate output buffers between executions.
    void bind(ObjectId id, DeviceTensor t);
    /// Global rows [first_row, first_row + rows) of image `id` from / to host
    /// memory (`pitch` bytes per host row); must lie inside the band storage.
    void upload_rows(ObjectId id, const void* host, std::size_t pitch, int first_row, int rows, int frame = 0);
    void download_rows(ObjectId id, void* host, std::size_t pitch, int first_row, int rows, int frame = 0);
    /// Enqueue one execution (halo exchanges + all groups, all frames).
    void launch();
    void synchronize();
    /// End to end from host memory, frame 0, single-group programs: `src` holds
    /// the input slab rows [src_row0, src_row1), `dst` receives output rows
    /// [row0, row1) of `output`.  Pieces of `piece_rows` output rows are
    /// pipelined over three streams (upload of piece i+1, kernel of piece i,
    /// download of piece i-1).  Returns when `dst` is complete.  Page-locked
    /// host memory (gvxb_host_alloc / gvxb_host_register) DMAs at full rate.
    void run_host(const void* src, std::size_t src_pitch, ObjectId output, void* dst, std::size_t dst_pitch,
                  int piece_rows = 1024);
    /// Packed host rows of one image (W * bytes-per-pixel per row): the
    /// input slab's rows, or an output's band rows.  Pageable memory is
    /// staged through page-locked slots; `drain` (outputs with page-locked
    /// `host` only) receives a copy of each piece as soon as it has landed.
    struct HostRows {
        ObjectId id = kInvalidId;
        void* host = nullptr;
        bool page_locked = false;
        void* drain = nullptr;
    };
    /// As run_host for the program's single input and any of its image
    /// outputs, with pageable or page-locked host rows (host copies of one
    /// piece overlap the transfers and kernel of the others).  Returns the
    /// device-counted pixel reads of the execution.
    long long run_host_rows(const HostRows& input, const std::vector<HostRows>& outputs, int piece_rows = 1024);
    int launches_per_run() const;
    std::string describe() const;

    struct Impl;

private:
    friend class BandGroup;
    friend struct detail::BandAccess;
    BandedSession();
    std::unique_ptr<Impl> impl_;
};

/// `devices.size()` bands of one image driven from one process: band g runs
/// on devices[g] (entries may repeat: several bands on one GPU), halo rows
/// move as strided peer copies (NVLink P2P between GPUs) on an exchange
/// stream, ordered by events, overlapping the interior rows.
class BandGroup {
public:
    BandGroup(const OptimizedPlan& plan, const std::vector<int>& devices, int frames = 1);
    ~BandGroup();
    BandGroup(const BandGroup&) = delete;
    BandGroup& operator=(const BandGroup&) = delete;
    int size() const;
    BandedSession& band(int g);
    void launch();
    void synchronize();

private:
    std::vector<std::unique_ptr<BandedSession>> bands_;
};

/// Number of CUDA devices visible (0 on a host without GPUs).
int device_count();

} // namespace gvx
