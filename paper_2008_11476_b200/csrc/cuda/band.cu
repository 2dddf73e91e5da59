// Row bands across GPUs (include/gvxb.h "multi-GPU row bands"): the band
// plan (rows, overlap split, exchange schedule), strided peer copies for
// bands driven from one process, and the NCCL halo exchange between
// processes (one rank per GPU, NVLink / NVSwitch).
//
// No reference counterpart: the reference splits rows over <= 4 host
// threads of one process (ref:src/execute.cpp:392-419).  SURVEY.md §8e.
//
// NCCL is resolved at first use with dlopen("libnccl.so.2") so this library
// still loads (and the CPU suite checks its symbols) where NCCL or a driver
// is absent; in a process that already loaded torch's NCCL the same soname
// resolves to that copy.
#include "common.cuh"

#include <nccl.h>

#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

using namespace gvxb_impl;

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("cannot load NCCL: ") + (e ? e : "libnccl.so.2 not found");
            return;
        }
        auto sym = [&](const char* name, auto& fn) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        api.ok = sym("ncclGetUniqueId", api.get_unique_id) && sym("ncclCommInitRank", api.comm_init_rank) &&
                 sym("ncclCommDestroy", api.comm_destroy) && sym("ncclSend", api.send) &&
                 sym("ncclRecv", api.recv) && sym("ncclGroupStart", api.group_start) &&
                 sym("ncclGroupEnd", api.group_end) && sym("ncclAllReduce", api.all_reduce) &&
                 sym("ncclGetErrorString", api.error_string);
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
    return fail(GVXB_ERR_CUDA, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

} // namespace

struct gvxb_comm_s {
    int device = 0, rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;   // exchange stream (overlaps the compute stream)
    cudaEvent_t ready = nullptr;     // compute stream -> exchange stream
    cudaEvent_t done = nullptr;      // exchange stream -> compute stream
    double* scratch = nullptr;       // all-reduce value (device)
    bool posted = false;
};

extern "C" {

int gvxb_band_rows(int32_t h, int32_t world, int32_t rank, int32_t* row0, int32_t* row1) {
    if (world < 1 || rank < 0 || rank >= world || h < 0) return fail(GVXB_ERR_INVALID, "bad band query");
    const int64_t base = h / world, extra = h % world;
    *row0 = static_cast<int32_t>(rank * base + (rank < extra ? rank : extra));
    *row1 = static_cast<int32_t>(*row0 + base + (rank < extra ? 1 : 0));
    return GVXB_OK;
}

int gvxb_band_plan_make(int32_t h, int32_t world, int32_t rank, int32_t halo, gvxb_band_plan* p) {
    if (!p || halo < 0) return fail(GVXB_ERR_INVALID, "bad band plan query");
    std::memset(p, 0, sizeof(*p));
    if (int rc = gvxb_band_rows(h, world, rank, &p->row0, &p->row1)) return rc;
    if (world > 1 && h / world < halo)
        return fail(GVXB_ERR_INVALID, "bands of " + std::to_string(h / world) + " rows are thinner than the halo (" +
                                          std::to_string(halo) + "): use fewer bands");
    p->height = h;
    p->world = world;
    p->rank = rank;
    p->halo = halo;
    p->src_row0 = std::max(0, p->row0 - halo);
    p->src_row1 = std::min(h, p->row1 + halo);
    // interior rows read source rows [r - halo, r + halo] that this band owns
    // (or that lie outside the image: those clamp into owned rows)
    const int32_t lo = rank > 0 ? p->row0 + halo : p->row0;
    const int32_t hi = rank < world - 1 ? p->row1 - halo : p->row1;
    if (lo < hi) {
        p->interior_row0 = lo;
        p->interior_row1 = hi;
        if (lo > p->row0) p->edge_row0[p->n_edges] = p->row0, p->edge_row1[p->n_edges++] = lo;
        if (hi < p->row1) p->edge_row0[p->n_edges] = hi, p->edge_row1[p->n_edges++] = p->row1;
    } else {
        p->interior_row0 = p->interior_row1 = p->row0;
        if (p->row1 > p->row0) p->edge_row0[0] = p->row0, p->edge_row1[0] = p->row1, p->n_edges = 1;
    }
    p->peer[0] = p->peer[1] = -1;
    if (rank > 0 && p->row0 > p->src_row0) { // upper neighbour: its last rows <-> my first rows
        p->peer[0] = rank - 1;
        p->recv_row0[0] = p->src_row0;
        p->recv_rows[0] = p->row0 - p->src_row0;
        p->send_row0[0] = p->row0;
        p->send_rows[0] = std::min(halo, p->row1 - p->row0);
    }
    if (rank < world - 1 && p->src_row1 > p->row1) {
        p->peer[1] = rank + 1;
        p->recv_row0[1] = p->row1;
        p->recv_rows[1] = p->src_row1 - p->row1;
        p->send_rows[1] = std::min(halo, p->row1 - p->row0);
        p->send_row0[1] = p->row1 - p->send_rows[1];
    }
    return GVXB_OK;
}

int gvxb_enable_peer(gvxb_ctx ctx, int peer) {
    if (peer == ctx->device) return GVXB_OK;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, ctx->device, peer);
    if (!can) return fail(GVXB_ERR_UNSUPPORTED, "peer access not possible");
    cudaSetDevice(ctx->device);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return GVXB_OK;
    }
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaDeviceEnablePeerAccess");
}

int gvxb_copy_peer_rows(gvxb_ctx ctx, void* dst, size_t dpitch, int dst_dev, const void* src, size_t spitch,
                        int src_dev, size_t row_bytes, size_t rows) {
    gvxb_impl::untracked_op(ctx);
    if (!rows || !row_bytes) return GVXB_OK;
    cudaError_t e;
    if (dst_dev == src_dev) {
        e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, cudaMemcpyDeviceToDevice, ctx->stream);
        return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaMemcpy2DAsync (rows)");
    }
    // one strided DMA for the whole row block (not one submission per row)
    cudaMemcpy3DPeerParms pp{};
    pp.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), spitch, row_bytes, rows);
    pp.srcDevice = src_dev;
    pp.dstPtr = make_cudaPitchedPtr(dst, dpitch, row_bytes, rows);
    pp.dstDevice = dst_dev;
    pp.extent = make_cudaExtent(row_bytes, rows, 1);
    e = cudaMemcpy3DPeerAsync(&pp, ctx->stream);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaMemcpy3DPeerAsync (rows)");
}

int gvxb_stream_wait_event(gvxb_ctx ctx, void* ev) {
    gvxb_impl::untracked_op(ctx);
    cudaError_t e = cudaStreamWaitEvent(ctx->stream, static_cast<cudaEvent_t>(ev), 0);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaStreamWaitEvent");
}

// ---------------------------------------------------------------- NCCL

int gvxb_comm_available(void) { return nccl().ok ? 1 : 0; }

int gvxb_comm_unique_id(uint8_t id[GVXB_COMM_ID_BYTES]) {
    static_assert(sizeof(ncclUniqueId) == GVXB_COMM_ID_BYTES, "ncclUniqueId size");
    if (!nccl().ok) return fail(GVXB_ERR_UNSUPPORTED, nccl().why);
    ncclUniqueId u;
    if (ncclResult_t r = nccl().get_unique_id(&u)) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
    return GVXB_OK;
}

int gvxb_comm_create(int device, int rank, int world, const uint8_t id[GVXB_COMM_ID_BYTES], gvxb_comm* out) {
    if (!nccl().ok) return fail(GVXB_ERR_UNSUPPORTED, nccl().why);
    if (world < 1 || rank < 0 || rank >= world) return fail(GVXB_ERR_INVALID, "bad rank / world");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    auto* c = new gvxb_comm_s();
    c->device = device;
    c->rank = rank;
    c->world = world;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    if (ncclResult_t r = nccl().comm_init_rank(&c->comm, world, u, rank)) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaMalloc(&c->scratch, sizeof(double))) != cudaSuccess) {
        gvxb_comm_destroy(c);
        return cuda_fail(e, "communicator resources");
    }
    *out = c;
    return GVXB_OK;
}

int gvxb_comm_destroy(gvxb_comm c) {
    if (!c) return GVXB_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm) nccl().comm_destroy(c->comm);
    if (c->scratch) cudaFree(c->scratch);
    if (c->ready) cudaEventDestroy(c->ready);
    if (c->done) cudaEventDestroy(c->done);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return GVXB_OK;
}

int gvxb_halo_start(gvxb_ctx ctx, gvxb_comm c, const gvxb_band_plan* p, const gvxb_image* slab) {
    gvxb_impl::untracked_op(ctx);
    if (!c || !p || !slab) return fail(GVXB_ERR_INVALID, "halo exchange: null argument");
    if (p->world != c->world || p->rank != c->rank) return fail(GVXB_ERR_INVALID, "band plan / communicator mismatch");
    cudaError_t e = cudaEventRecord(c->ready, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, c->ready, 0);
    if (e != cudaSuccess) return cuda_fail(e, "halo exchange ordering");
    if (p->world > 1 && (p->peer[0] >= 0 || p->peer[1] >= 0)) {
        const int frames = std::max(1, slab->frames);
        const int64_t fstride = slab->frames > 1 ? slab->frame_stride : 0;
        auto* base = static_cast<uint8_t*>(slab->data);
        auto row = [&](int f, int32_t r) { return base + f * fstride + static_cast<int64_t>(r - p->src_row0) * slab->pitch; };
        if (ncclResult_t r = nccl().group_start()) return nccl_fail(r, "ncclGroupStart");
        for (int f = 0; f < frames; ++f)
            for (int s = 0; s < 2; ++s) {
                if (p->peer[s] < 0) continue;
                // rows are `pitch` apart and contiguous: one message per side
                // (both ranks allocate the object with the same pitch)
                ncclResult_t r = nccl().send(row(f, p->send_row0[s]), static_cast<size_t>(p->send_rows[s]) * slab->pitch,
                                             ncclUint8, p->peer[s], c->comm, c->stream);
                if (r == ncclSuccess)
                    r = nccl().recv(row(f, p->recv_row0[s]), static_cast<size_t>(p->recv_rows[s]) * slab->pitch,
                                    ncclUint8, p->peer[s], c->comm, c->stream);
                if (r != ncclSuccess) {
                    nccl().group_end();
                    return nccl_fail(r, "ncclSend/ncclRecv");
                }
            }
        if (ncclResult_t r = nccl().group_end()) return nccl_fail(r, "ncclGroupEnd");
    }
    e = cudaEventRecord(c->done, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "halo exchange event");
    c->posted = true;
    return GVXB_OK;
}

int gvxb_halo_wait(gvxb_ctx ctx, gvxb_comm c) {
    gvxb_impl::untracked_op(ctx);
    if (!c) return fail(GVXB_ERR_INVALID, "halo wait: null communicator");
    if (!c->posted) return GVXB_OK;
    cudaError_t e = cudaStreamWaitEvent(ctx->stream, c->done, 0);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "halo wait");
}

int gvxb_comm_allreduce_max(gvxb_comm c, double* value) {
    if (!c || !value) return fail(GVXB_ERR_INVALID, "all-reduce: null argument");
    cudaSetDevice(c->device);
    cudaError_t e = cudaMemcpyAsync(c->scratch, value, sizeof(double), cudaMemcpyHostToDevice, c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "all-reduce upload");
    if (ncclResult_t r = nccl().all_reduce(c->scratch, c->scratch, 1, ncclFloat64, ncclMax, c->comm, c->stream))
        return nccl_fail(r, "ncclAllReduce");
    e = cudaMemcpyAsync(value, c->scratch, sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "all-reduce download");
}

int gvxb_comm_barrier(gvxb_comm c) {
    double v = 0.0;
    return gvxb_comm_allreduce_max(c, &v);
}

} // extern "C"
