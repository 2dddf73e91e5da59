// Device runtime behind the C-ABI (include/gvxb.h): contexts, streams,
// memory, copies, events, status word, NVRTC JIT and peer access.
//
// Driver-API symbols (module loading, launches) are resolved at run time via
// cudaGetDriverEntryPoint so this library loads on a machine without a GPU
// driver (the CPU test suite checks the exported symbols there).
#include "common.cuh"

#include <atomic>

#include <cuda.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace gvxb_impl {

thread_local std::string g_last_error;
thread_local std::string g_jit_log;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(GVXB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

std::atomic<long long> g_total_launches{0}; // every context's launches

int check_launch(gvxb_ctx ctx, const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    ++ctx->launches;
    ++g_total_launches;
    return GVXB_OK;
}

namespace {
bool overlaps(const gvxb_range& a, const gvxb_range& b) { return a.lo < b.hi && b.lo < a.hi && a.lo < a.hi && b.lo < b.hi; }
} // namespace

int pdl_must_wait(gvxb_ctx ctx, const gvxb_range* r, int nr, const gvxb_range* w, int nw) {
    if (!ctx->prev_kernel) return 1;
    for (int i = 0; i < nr; ++i)
        for (int k = 0; k < ctx->prev_nw; ++k)
            if (overlaps(r[i], ctx->prev_w[k])) return 1; // RAW
    for (int i = 0; i < nw; ++i) {
        for (int k = 0; k < ctx->prev_nw; ++k)
            if (overlaps(w[i], ctx->prev_w[k])) return 1; // WAW
        for (int k = 0; k < ctx->prev_nr; ++k)
            if (overlaps(w[i], ctx->prev_r[k])) return 1; // WAR
    }
    return 0;
}

namespace {
int nonempty(const gvxb_range* a, int n) {
    int k = 0;
    for (int i = 0; i < n; ++i) k += a[i].lo < a[i].hi ? 1 : 0;
    return k;
}
} // namespace

bool launch_overlaps(gvxb_ctx ctx, const gvxb_range* r, int nr, const gvxb_range* w, int nw) {
    const bool allowed = ctx->overlap > 0 || (ctx->overlap < 0 && ctx->stream == ctx->own_stream);
    return allowed && ctx->prev_kernel && !pdl_must_wait(ctx, r, nr, w, nw) &&
           ctx->prev_nr + nonempty(r, nr) <= kTrackedRanges && ctx->prev_nw + nonempty(w, nw) <= kTrackedRanges;
}

/// A launch independent of every kernel in the window overlaps them
/// (programmatic dependent launch, pdl_wait = 0) and joins the window; a
/// launch that depends on a one-kernel window overlaps its tail and waits
/// for it in the kernel (pdl_wait = 1); any other launch is fully
/// stream-ordered (it starts after all earlier work completed; its
/// griddepcontrol.wait is a no-op).  The last two start a new window.
int launch_tracked(gvxb_ctx ctx, const void* fn, dim3 grid, dim3 block, void** args, size_t smem,
                   const gvxb_range* r, int nr, const gvxb_range* w, int nw, const char* what) {
    const bool allowed = ctx->overlap > 0 || (ctx->overlap < 0 && ctx->stream == ctx->own_stream);
    const bool joins = launch_overlaps(ctx, r, nr, w, nw);
    // dependent on a one-kernel window: overlap its tail and wait for it in
    // the kernel (the caller passed pdl_wait = 1); the window restarts here
    const bool waits = !joins && allowed && ctx->prev_kernel && ctx->prev_launches == 1;
    const bool pdl = joins || waits;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    if (pdl) {
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return cuda_fail(e, what);
    if (!joins) ctx->prev_nr = ctx->prev_nw = ctx->prev_launches = 0; // a new window
    if (ctx->prev_nr + nonempty(r, nr) <= kTrackedRanges && ctx->prev_nw + nonempty(w, nw) <= kTrackedRanges) {
        for (int i = 0; i < nr; ++i)
            if (r[i].lo < r[i].hi) ctx->prev_r[ctx->prev_nr++] = r[i];
        for (int i = 0; i < nw; ++i)
            if (w[i].lo < w[i].hi) ctx->prev_w[ctx->prev_nw++] = w[i];
        ctx->prev_launches += 1;
        ctx->prev_kernel = true;
    } else {
        ctx->prev_kernel = false; // untrackable: the next launch is stream-ordered
    }
    return check_launch(ctx, what);
}

} // namespace gvxb_impl

using namespace gvxb_impl;

struct gvxb_module_s {
    CUmodule module = nullptr;
    std::vector<CUfunction> functions;
};

namespace {

struct DriverApi {
    CUresult (*module_load_data)(CUmodule*, const void*) = nullptr;
    CUresult (*module_unload)(CUmodule) = nullptr;
    CUresult (*module_get_function)(CUfunction*, CUmodule, const char*) = nullptr;
    CUresult (*launch_kernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                              unsigned, CUstream, void**, void**) = nullptr;
    CUresult (*func_set_attribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    bool ok = false;
};

DriverApi& driver() {
    static DriverApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn != nullptr;
        };
        api.ok = get("cuModuleLoadData", reinterpret_cast<void**>(&api.module_load_data)) &&
                 get("cuModuleUnload", reinterpret_cast<void**>(&api.module_unload)) &&
                 get("cuModuleGetFunction", reinterpret_cast<void**>(&api.module_get_function)) &&
                 get("cuLaunchKernel", reinterpret_cast<void**>(&api.launch_kernel)) &&
                 get("cuFuncSetAttribute", reinterpret_cast<void**>(&api.func_set_attribute));
    });
    return api;
}

} // namespace

extern "C" {

const char* gvxb_last_error(void) { return g_last_error.c_str(); }
int gvxb_abi_version(void) { return GVXB_ABI_VERSION; }

int gvxb_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
        return fail(GVXB_ERR_NO_DEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
    }
    *count = n;
    return GVXB_OK;
}

int gvxb_ctx_create(int device, gvxb_ctx* out) {
    int n = 0;
    if (int rc = gvxb_device_count(&n)) return rc;
    if (device < 0 || device >= n) return fail(GVXB_ERR_NO_DEVICE, "device index out of range");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    auto* c = new gvxb_ctx_s();
    c->device = device;
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaStreamCreate");
    }
    c->stream = c->own_stream;
    e = cudaMalloc(&c->status, sizeof(unsigned) + sizeof(unsigned long long) * 2);
    if (e != cudaSuccess) {
        cudaStreamDestroy(c->own_stream);
        delete c;
        return cuda_fail(e, "cudaMalloc(status)");
    }
    c->counter = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(c->status) + 8);
    cudaMemset(c->status, 0, sizeof(unsigned) + sizeof(unsigned long long) * 2);
    *out = c;
    return GVXB_OK;
}

int gvxb_ctx_destroy(gvxb_ctx ctx) {
    if (!ctx) return GVXB_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->status);
    cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return GVXB_OK;
}

int gvxb_ctx_set_overlap(gvxb_ctx ctx, int mode) {
    ctx->overlap = mode < 0 ? -1 : (mode > 0 ? 1 : 0);
    untracked_op(ctx);
    return GVXB_OK;
}

int gvxb_ctx_set_stream(gvxb_ctx ctx, void* s) {
    cudaStream_t to = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
    if (to != ctx->stream) untracked_op(ctx);
    ctx->stream = to;
    return GVXB_OK;
}

void* gvxb_ctx_stream(gvxb_ctx ctx) { return ctx->stream; }
int gvxb_ctx_device(gvxb_ctx ctx) { return ctx->device; }
int gvxb_ctx_sm_count(gvxb_ctx ctx) { return ctx->sm_count; }
int64_t gvxb_launch_count(gvxb_ctx ctx) { return ctx->launches; }
int64_t gvxb_total_launch_count(void) { return g_total_launches.load(); }

int gvxb_sync(gvxb_ctx ctx) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaStreamSynchronize");
}

// GVX_GUARD_ALLOC=1 (debugging; compute-sanitizer stand-in): every
// allocation is framed by kGuard bytes of 0xA5 on both sides; gvxb_free
// synchronizes the device and checks them, counting (and reporting on
// stderr) each allocation whose guards a kernel overwrote.
namespace {
constexpr size_t kGuard = 4096;
constexpr unsigned char kGuardByte = 0xA5;
struct GuardedAlloc {
    void* base;
    size_t bytes;
};
std::mutex g_guard_mu;
std::vector<std::pair<void*, GuardedAlloc>> g_guarded;
std::atomic<long long> g_guard_violations{0};
bool guard_mode() {
    static const bool on = [] {
        const char* e = std::getenv("GVX_GUARD_ALLOC");
        return e && *e && *e != '0';
    }();
    return on;
}
bool guards_intact(const GuardedAlloc& g) {
    std::vector<unsigned char> h(kGuard);
    const unsigned char* base = static_cast<const unsigned char*>(g.base);
    for (const unsigned char* at : {base, base + kGuard + g.bytes}) {
        if (cudaMemcpy(h.data(), at, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
        for (unsigned char b : h)
            if (b != kGuardByte) return false;
    }
    return true;
}
} // namespace

int gvxb_alloc(gvxb_ctx ctx, size_t bytes, void** p) {
    cudaSetDevice(ctx->device);
    if (guard_mode()) {
        const size_t n = (bytes ? bytes : 16), padded = (n + 255) & ~size_t(255);
        void* base = nullptr;
        cudaError_t e = cudaMalloc(&base, padded + 2 * kGuard);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
        if ((e = cudaMemset(base, kGuardByte, padded + 2 * kGuard)) != cudaSuccess ||
            (e = cudaDeviceSynchronize()) != cudaSuccess)
            return cuda_fail(e, "guard fill");
        *p = static_cast<char*>(base) + kGuard;
        std::lock_guard<std::mutex> lk(g_guard_mu);
        g_guarded.push_back({*p, GuardedAlloc{base, padded}});
        return GVXB_OK;
    }
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaMalloc");
}

int gvxb_free(gvxb_ctx ctx, void* p) {
    cudaSetDevice(ctx->device);
    if (guard_mode() && p) {
        GuardedAlloc g{nullptr, 0};
        {
            std::lock_guard<std::mutex> lk(g_guard_mu);
            for (auto it = g_guarded.begin(); it != g_guarded.end(); ++it)
                if (it->first == p) {
                    g = it->second;
                    g_guarded.erase(it);
                    break;
                }
        }
        if (g.base) {
            cudaDeviceSynchronize();
            if (!guards_intact(g)) {
                ++g_guard_violations;
                std::fprintf(stderr, "gvxb: guard bytes around a %zu-byte allocation at %p overwritten\n", g.bytes, p);
            }
            cudaError_t e = cudaFree(g.base);
            return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaFree");
        }
    }
    cudaError_t e = cudaFree(p);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaFree");
}

int64_t gvxb_guard_check(int* live) {
    long long bad = g_guard_violations.load();
    std::lock_guard<std::mutex> lk(g_guard_mu);
    if (!g_guarded.empty()) cudaDeviceSynchronize();
    for (const auto& a : g_guarded)
        if (!guards_intact(a.second)) ++bad;
    if (live) *live = static_cast<int>(g_guarded.size());
    return bad;
}

int gvxb_host_alloc(size_t bytes, void** p) {
    cudaError_t e = cudaHostAlloc(p, bytes ? bytes : 16, cudaHostAllocPortable);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaHostAlloc");
}

int gvxb_host_free(void* p) {
    cudaError_t e = cudaFreeHost(p);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaFreeHost");
}

int gvxb_host_register(void* p, size_t bytes) {
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaHostRegister");
}

int gvxb_host_unregister(void* p) {
    cudaError_t e = cudaHostUnregister(p);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaHostUnregister");
}

int gvxb_host_is_pinned(const void* p, int* pinned) {
    cudaPointerAttributes a{};
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError(); // unregistered pageable memory on older drivers
        *pinned = 0;
        return GVXB_OK;
    }
    *pinned = a.type == cudaMemoryTypeHost ? 1 : 0;
    return GVXB_OK;
}

int gvxb_memset(gvxb_ctx ctx, void* p, int v, size_t bytes) {
    untracked_op(ctx);
    cudaError_t e = cudaMemsetAsync(p, v, bytes, ctx->stream);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaMemsetAsync");
}

int gvxb_upload_2d(gvxb_ctx ctx, void* dst, size_t dpitch, const void* src, size_t spitch,
                   size_t row_bytes, size_t rows) {
    untracked_op(ctx);
    if (!rows || !row_bytes) return GVXB_OK;
    // dense on both sides: one linear copy (the DMA engines stream it faster)
    cudaError_t e = dpitch == row_bytes && spitch == row_bytes
                        ? cudaMemcpyAsync(dst, src, row_bytes * rows, cudaMemcpyHostToDevice, ctx->stream)
                        : cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, cudaMemcpyHostToDevice,
                                            ctx->stream);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaMemcpy2DAsync(H2D)");
}

int gvxb_download_2d(gvxb_ctx ctx, void* dst, size_t dpitch, const void* src, size_t spitch,
                     size_t row_bytes, size_t rows) {
    untracked_op(ctx);
    if (!rows || !row_bytes) return GVXB_OK;
    cudaError_t e = dpitch == row_bytes && spitch == row_bytes
                        ? cudaMemcpyAsync(dst, src, row_bytes * rows, cudaMemcpyDeviceToHost, ctx->stream)
                        : cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, cudaMemcpyDeviceToHost,
                                            ctx->stream);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaMemcpy2DAsync(D2H)");
}

int gvxb_copy_d2d(gvxb_ctx ctx, void* dst, const void* src, size_t bytes) {
    untracked_op(ctx);
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "cudaMemcpyAsync(D2D)");
}

int gvxb_event_create(void** ev) {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreate(&e);
    *ev = e;
    return r == cudaSuccess ? GVXB_OK : cuda_fail(r, "cudaEventCreate");
}

int gvxb_event_destroy(void* ev) {
    cudaEventDestroy(static_cast<cudaEvent_t>(ev));
    return GVXB_OK;
}

int gvxb_event_record(gvxb_ctx ctx, void* ev) {
    untracked_op(ctx);
    cudaError_t r = cudaEventRecord(static_cast<cudaEvent_t>(ev), ctx->stream);
    return r == cudaSuccess ? GVXB_OK : cuda_fail(r, "cudaEventRecord");
}

int gvxb_event_elapsed_ms(void* a, void* b, float* ms) {
    cudaError_t r = cudaEventSynchronize(static_cast<cudaEvent_t>(b));
    if (r != cudaSuccess) return cuda_fail(r, "cudaEventSynchronize");
    r = cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b));
    return r == cudaSuccess ? GVXB_OK : cuda_fail(r, "cudaEventElapsedTime");
}

int gvxb_event_sync(void* ev) {
    cudaError_t r = cudaEventSynchronize(static_cast<cudaEvent_t>(ev));
    return r == cudaSuccess ? GVXB_OK : cuda_fail(r, "cudaEventSynchronize");
}

int gvxb_status_reset(gvxb_ctx ctx) {
    untracked_op(ctx);
    cudaError_t e = cudaMemsetAsync(ctx->status, 0, sizeof(unsigned) + 2 * sizeof(unsigned long long),
                                    ctx->stream);
    return e == cudaSuccess ? GVXB_OK : cuda_fail(e, "status reset");
}

int gvxb_status_read(gvxb_ctx ctx, uint32_t* status) {
    unsigned v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, ctx->status, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "status read");
    *status = v;
    return GVXB_OK;
}

int gvxb_status_ptr(gvxb_ctx ctx, uint32_t** p) {
    *p = ctx->status;
    return GVXB_OK;
}

int gvxb_counter_ptr(gvxb_ctx ctx, unsigned long long** p) {
    *p = ctx->counter;
    return GVXB_OK;
}

int gvxb_status_counter_read(gvxb_ctx ctx, uint32_t* status, long long* counter) {
    // status word at +0, counter at +8 of the same allocation
    unsigned long long v[2] = {0, 0};
    cudaError_t e = cudaMemcpyAsync(v, ctx->status, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "status read");
    *status = static_cast<uint32_t>(v[0] & 0xFFFFFFFFu);
    *counter = static_cast<long long>(v[1]);
    return GVXB_OK;
}

int gvxb_counter_read(gvxb_ctx ctx, long long* reads) {
    unsigned long long v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, ctx->counter, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "counter read");
    *reads = static_cast<long long>(v);
    return GVXB_OK;
}

// ---------------------------------------------------------------------- JIT

const char* gvxb_jit_log(void) { return g_jit_log.c_str(); }

int gvxb_jit_build(gvxb_ctx ctx, const char* source, const char* const* names, int n, gvxb_module* out) {
    DriverApi& drv = driver();
    if (!drv.ok) return fail(GVXB_ERR_NO_DEVICE, "CUDA driver entry points unavailable");
    cudaSetDevice(ctx->device);
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, ctx->device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, ctx->device);
    if (major != 10) return fail(GVXB_ERR_UNSUPPORTED, "graphvx-b200 kernels target sm_100a (B200)");

    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, source, "gvx_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
        return fail(GVXB_ERR_NVRTC, "nvrtcCreateProgram failed");
    const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17",
                          "--device-as-default-execution-space", "-lineinfo"};
    nvrtcResult r = nvrtcCompileProgram(prog, 5, opts);
    size_t log_size = 0;
    nvrtcGetProgramLogSize(prog, &log_size);
    g_jit_log.assign(log_size, '\0');
    if (log_size) nvrtcGetProgramLog(prog, &g_jit_log[0]);
    if (r != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        return fail(GVXB_ERR_NVRTC, std::string("NVRTC compile failed: ") + g_jit_log.substr(0, 2000));
    }
    size_t cubin_size = 0;
    nvrtcGetCUBINSize(prog, &cubin_size);
    std::vector<char> cubin(cubin_size);
    nvrtcGetCUBIN(prog, cubin.data());
    std::vector<std::string> lowered(names, names + n); // extern "C" kernels: unmangled
    nvrtcDestroyProgram(&prog);

    auto* m = new gvxb_module_s();
    if (drv.module_load_data(&m->module, cubin.data()) != CUDA_SUCCESS) {
        delete m;
        return fail(GVXB_ERR_CUDA, "cuModuleLoadData failed");
    }
    for (const std::string& ln : lowered) {
        CUfunction f = nullptr;
        if (drv.module_get_function(&f, m->module, ln.c_str()) != CUDA_SUCCESS) {
            drv.module_unload(m->module);
            delete m;
            return fail(GVXB_ERR_CUDA, "cuModuleGetFunction(" + ln + ") failed");
        }
        drv.func_set_attribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 200 * 1024);
        m->functions.push_back(f);
    }
    *out = m;
    return GVXB_OK;
}

int gvxb_jit_free(gvxb_module m) {
    if (!m) return GVXB_OK;
    if (driver().ok && m->module) driver().module_unload(m->module);
    delete m;
    return GVXB_OK;
}

int gvxb_jit_launch(gvxb_ctx ctx, gvxb_module m, int k, const unsigned grid[3], const unsigned block[3],
                    size_t smem, void** args) {
    untracked_op(ctx);
    if (k < 0 || k >= static_cast<int>(m->functions.size())) return fail(GVXB_ERR_INVALID, "bad kernel index");
    if (grid[0] == 0 || grid[1] == 0 || grid[2] == 0) return GVXB_OK;
    CUresult r = driver().launch_kernel(m->functions[static_cast<std::size_t>(k)], grid[0], grid[1], grid[2],
                                        block[0], block[1], block[2], static_cast<unsigned>(smem),
                                        static_cast<CUstream>(ctx->stream), args, nullptr);
    if (r != CUDA_SUCCESS) return fail(GVXB_ERR_CUDA, "cuLaunchKernel failed (" + std::to_string(r) + ")");
    ++ctx->launches;
    ++g_total_launches;
    return GVXB_OK;
}

} // extern "C"
