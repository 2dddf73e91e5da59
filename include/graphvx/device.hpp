// graphvx-b200 — additive device-resident execution API (not in the
// reference).  run_plan / run_naive keep the reference's host-Buffer
// contract; DeviceSession launches the same lowered program on device
// buffers the caller owns (frame batches, benchmarks, multi-GPU bands) with
// no host copies on the critical path.
#pragma once

#include "graphvx/execute.hpp"

#include <memory>
#include <string>

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

/// Number of CUDA devices visible (0 on a host without GPUs).
int device_count();

} // namespace gvx
