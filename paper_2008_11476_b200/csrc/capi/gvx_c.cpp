// C facade over the public C++ API (include/gvx_c.h).
#include "gvx_c.h"

#include "../configs/config_graphs.hpp"
#include "../configs/json_runner.hpp"
#include "graphvx/device.hpp"
#include "graphvx/optimize.hpp"
#include "hostcopy.hpp"
#include "program.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <set>
#include <string>

namespace {

thread_local std::string g_err;

int fail_from(const std::exception& e) {
    g_err = e.what();
    if (auto* ge = dynamic_cast<const gvx::Error*>(&e)) return static_cast<int>(ge->code()) + 1;
    return 100;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        return fail_from(e);
    }
}

} // namespace

struct gvxc_graph_s {
    int cfg = 0;
    int width = 0, height = 0;
    gvx::Context ctx;
    gvx_configs::ConfigGraph cg;
    gvx::VerifiedGraph impl;
    gvx::OptimizedPlan plan;
    gvx::Buffer input; ///< reused between host runs, page-locked once
    /// page-locked output vectors handed back to the engine before each run
    /// (detail::run_*_pooled): outputs DMA straight into them
    std::map<gvx::ObjectId, std::vector<std::uint8_t>> pool;
    gvx::ExecutionReport last; ///< outputs of the latest host run (output_ptr)
    std::set<const void*> registered;

    void pin(const std::vector<std::uint8_t>& v) {
        if (v.size() < (1u << 20) || registered.count(v.data())) return;
        if (gvxb_host_register(const_cast<std::uint8_t*>(v.data()), v.size()) == GVXB_OK) registered.insert(v.data());
    }
    ~gvxc_graph_s() {
        for (const void* p : registered) gvxb_host_unregister(const_cast<void*>(p));
    }
};

struct gvxc_session_s {
    gvxc_graph g = nullptr;
    std::unique_ptr<gvx::DeviceSession> s;
};

extern "C" {

const char* gvxc_last_error(void) { return g_err.c_str(); }
int gvxc_device_count(void) { return gvx::device_count(); }

int gvxc_config_create(int cfg, int w, int h, int virtual_mid, gvxc_graph* out) {
    return guarded([&] {
        auto g = std::make_unique<gvxc_graph_s>();
        g->cfg = cfg;
        g->width = w;
        g->height = h;
        g->cg = gvx_configs::build_config(g->ctx, cfg, w, h, virtual_mid != 0);
        g->impl = gvx_configs::verified_impl(g->ctx, *g->cg.graph);
        g->plan = gvx::optimize(g->impl, g->ctx);
        *out = g.release();
    });
}

int gvxc_graph_destroy(gvxc_graph g) {
    delete g;
    return 0;
}

int gvxc_graph_describe(gvxc_graph g, int naive, char* buf, size_t cap) {
    return guarded([&] {
        std::string d = naive ? gvx::DeviceSession(g->impl).describe() : gvx::DeviceSession(g->plan).describe();
        if (cap) {
            std::strncpy(buf, d.c_str(), cap - 1);
            buf[cap - 1] = '\0';
        }
    });
}

int gvxc_graph_pass_stats(gvxc_graph g, long long st[8]) {
    const gvx::PassStats& p = g->plan.stats;
    const long long v[8] = {p.nodes_before, p.nodes_alive, p.nodes_removed, p.transfers_naive,
                            p.transfers_optimized, p.fused_groups, p.launches_before, p.launches_after};
    std::memcpy(st, v, sizeof(v));
    return 0;
}

namespace {

void copy_outputs(gvxc_graph g, const std::map<gvx::ObjectId, gvx::Buffer>& outs, void* out, long long* hist,
                  double* stats) {
    if (g->cfg == 4) {
        const gvx::Buffer& hb = outs.at(g->cg.outputs[0]);
        if (hist)
            for (std::size_t i = 0; i < hb.dist.counts.size(); ++i) hist[i] = hb.dist.counts[i];
        if (stats) {
            stats[0] = outs.at(g->cg.outputs[1]).scalar.as_real();
            stats[1] = outs.at(g->cg.outputs[2]).scalar.as_real();
        }
        return;
    }
    const gvx::Buffer& b = outs.at(g->cg.outputs[0]);
    if (out) gvx::dev::parallel_copy(out, b.bytes.data(), b.bytes.size());
}

void ensure_input(gvxc_graph g) {
    if (!g->input.bytes.empty()) return;
    gvx::ResolvedDesc d;
    d.kind = gvx::ObjKind::Image;
    d.width = g->width;
    d.height = g->height;
    d.format = gvx::ImageFormat::U8;
    g->input = gvx::Buffer::image(d);
    g->input.id = g->cg.input;
    g->pin(g->input.bytes);
}

gvx::Buffer input_buffer(gvxc_graph g, const uint8_t* in) {
    gvx::ResolvedDesc d;
    d.kind = gvx::ObjKind::Image;
    d.width = g->width;
    d.height = g->height;
    d.format = gvx::ImageFormat::U8;
    gvx::Buffer b = gvx::Buffer::image(d);
    std::memcpy(b.bytes.data(), in, b.bytes.size());
    return b;
}

} // namespace

int gvxc_graph_run_host(gvxc_graph g, int naive, const uint8_t* in, void* out, long long* hist, double* stats,
                        long long counters[4]) {
    return guarded([&] {
        gvx::InputMap inputs;
        ensure_input(g);
        // in == the buffer from gvxc_graph_input_ptr: the caller filled it in place
        // the caller's frame goes into the page-locked input Buffer during the
        // upload, chunk by chunk (copy of chunk k+1 overlaps the DMA of chunk k)
        gvx::detail::HostFill fill;
        if (in && in != g->input.bytes.data()) {
            fill.id = g->cg.input;
            fill.src = in;
            if (!g->registered.count(g->input.bytes.data())) // not page-locked: copy up front
                gvx::dev::parallel_copy(g->input.bytes.data(), in, g->input.bytes.size()), fill.src = nullptr;
        }
        if (out && g->cfg != 4) { // the caller's destination may be filled piece by piece during the run
            fill.drain_id = g->cg.outputs.at(0);
            fill.drain_dst = out;
        }
        // recycle the previous run's (page-locked) output vectors
        for (auto& [id, b] : g->last.outputs)
            if (b.desc.kind == gvx::ObjKind::Image && !b.bytes.empty()) {
                g->pin(b.bytes);
                g->pool[id] = std::move(b.bytes);
            }
        g->last = gvx::ExecutionReport{};
        gvx::Buffer& slot = inputs[g->cg.input];
        slot = std::move(g->input);
        gvx::ExecutionReport r;
        try {
            r = naive ? gvx::detail::run_naive_pooled(g->impl, inputs, &g->pool, &fill)
                      : gvx::detail::run_plan_pooled(g->plan, inputs, &g->pool, &fill);
        } catch (...) {
            g->input = std::move(slot);
            throw;
        }
        g->input = std::move(slot);
        copy_outputs(g, r.outputs, fill.drained ? nullptr : out, hist, stats);
        if (counters) {
            counters[0] = r.counters.kernel_launches;
            counters[1] = r.counters.pixels_read;
            counters[2] = r.counters.pixels_written;
            counters[3] = r.counters.transfers_executed;
        }
        g->last = std::move(r);
    });
}

int gvxc_graph_input_ptr(gvxc_graph g, uint8_t** ptr, size_t* bytes) {
    return guarded([&] {
        ensure_input(g);
        *ptr = g->input.bytes.data();
        if (bytes) *bytes = g->input.bytes.size();
    });
}

int gvxc_graph_output_ptr(gvxc_graph g, const void** ptr, size_t* bytes) {
    return guarded([&] {
        auto it = g->last.outputs.find(g->cg.outputs.at(0));
        if (it == g->last.outputs.end() || it->second.desc.kind != gvx::ObjKind::Image)
            throw gvx::Error(gvx::ErrorCode::UnknownObject, "no image output from a previous host run");
        *ptr = it->second.bytes.data();
        if (bytes) *bytes = it->second.bytes.size();
    });
}

int gvxc_session_create(gvxc_graph g, int naive, int frames, gvxc_session* out) {
    return guarded([&] {
        auto s = std::make_unique<gvxc_session_s>();
        s->g = g;
        s->s = naive ? std::make_unique<gvx::DeviceSession>(g->impl, frames)
                     : std::make_unique<gvx::DeviceSession>(g->plan, frames);
        *out = s.release();
    });
}

int gvxc_session_destroy(gvxc_session s) {
    delete s;
    return 0;
}

namespace {
gvx::ObjectId slot_object(gvxc_session s, int slot) {
    if (slot == 0) return s->g->cg.input;
    const auto& outs = s->g->cg.outputs;
    if (slot < 1 || slot > static_cast<int>(outs.size())) throw gvx::Error(gvx::ErrorCode::UnknownObject, "bad slot");
    return outs[static_cast<std::size_t>(slot - 1)];
}
} // namespace

int gvxc_session_bind(gvxc_session s, int slot, void* dptr, int64_t pitch, int64_t fstride) {
    return guarded([&] { s->s->bind(slot_object(s, slot), gvx::DeviceTensor{dptr, pitch, fstride}); });
}

int gvxc_session_set_stream(gvxc_session s, void* stream) {
    return guarded([&] { s->s->set_stream(stream); });
}

int gvxc_session_set_overlap(gvxc_session s, int mode) {
    return guarded([&] { s->s->set_overlap(mode); });
}

int gvxc_session_launch(gvxc_session s) {
    return guarded([&] { s->s->launch(); });
}

int gvxc_session_sync(gvxc_session s) {
    return guarded([&] { s->s->synchronize(); });
}

int gvxc_session_launches(gvxc_session s) { return s->s->launches_per_run(); }

int gvxc_session_upload_input(gvxc_session s, int frame, const uint8_t* in) {
    return guarded([&] { s->s->upload(s->g->cg.input, input_buffer(s->g, in), frame); });
}

int gvxc_session_download(gvxc_session s, int slot, int frame, void* out, long long* hist, double* stats) {
    return guarded([&] {
        gvxc_graph g = s->g;
        std::map<gvx::ObjectId, gvx::Buffer> outs;
        if (g->cfg == 4) {
            for (gvx::ObjectId id : g->cg.outputs) outs[id] = s->s->download(id, frame);
        } else {
            const gvx::ObjectId id = slot_object(s, slot < 1 ? 1 : slot);
            outs[g->cg.outputs[0]] = s->s->download(id, frame);
        }
        copy_outputs(g, outs, out, hist, stats);
    });
}

long long gvxc_launch_count(void) {
    try {
        return gvx::dev::launch_count();
    } catch (...) {
        return -1;
    }
}

void* gvxc_default_stream(void) {
    try {
        return gvxb_ctx_stream(gvx::dev::context());
    } catch (...) {
        return nullptr;
    }
}

int gvxc_random_u8(int w, int h, unsigned long long seed, uint8_t* out) {
    return guarded([&] {
        gvx::ResolvedDesc d;
        d.kind = gvx::ObjKind::Image;
        d.width = w;
        d.height = h;
        d.format = gvx::ImageFormat::U8;
        gvx::Buffer b = gvx::random_buffer(d, seed);
        std::memcpy(out, b.bytes.data(), b.bytes.size());
    });
}

} // extern "C"

// ------------------------------------------------------------ pipelines

struct gvxc_pipeline_s {
    gvxc_graph g = nullptr;
    std::unique_ptr<gvx::HostPipeline> p;
    int depth = 1;
};

extern "C" {

int gvxc_pipeline_create(gvxc_graph g, int naive, int depth, gvxc_pipeline* out) {
    return guarded([&] {
        auto pl = std::make_unique<gvxc_pipeline_s>();
        pl->g = g;
        pl->depth = depth < 1 ? 1 : depth;
        pl->p = naive ? std::make_unique<gvx::HostPipeline>(g->impl, depth)
                      : std::make_unique<gvx::HostPipeline>(g->plan, depth);
        *out = pl.release();
    });
}

int gvxc_pipeline_destroy(gvxc_pipeline p) {
    delete p;
    return 0;
}

int gvxc_pipeline_submit(gvxc_pipeline p, const uint8_t* in) {
    return guarded([&] {
        p->p->submit(p->g->cg.input, in, static_cast<std::size_t>(p->g->width) * static_cast<std::size_t>(p->g->height));
    });
}

int gvxc_pipeline_submit_pinned(gvxc_pipeline p, const uint8_t* in) {
    return guarded([&] {
        p->p->submit_pinned(p->g->cg.input, in,
                            static_cast<std::size_t>(p->g->width) * static_cast<std::size_t>(p->g->height));
    });
}

int gvxc_host_register(void* ptr, size_t bytes) {
    return guarded([&] { gvx::dev::check(gvxb_host_register(ptr, bytes), "host register"); });
}

int gvxc_host_unregister(void* ptr) {
    return guarded([&] { gvx::dev::check(gvxb_host_unregister(ptr), "host unregister"); });
}

int gvxc_pipeline_pending(gvxc_pipeline p) { return p->p->pending(); }

int gvxc_pipeline_next_view(gvxc_pipeline p, const void** view, size_t* bytes, long long counters[4]) {
    return guarded([&] {
        gvxc_graph g = p->g;
        if (g->cfg == 4) throw gvx::Error(gvx::ErrorCode::UnknownObject, "config 4 has no image output");
        gvx::ExecutionReport r = p->p->next_view(g->cg.outputs.at(0), view);
        if (bytes)
            *bytes = (g->cfg == 1 || g->cfg == 5 ? 2u : 1u) * static_cast<std::size_t>(g->width) *
                     static_cast<std::size_t>(g->height);
        if (counters) {
            counters[0] = r.counters.kernel_launches;
            counters[1] = r.counters.pixels_read;
            counters[2] = r.counters.pixels_written;
            counters[3] = r.counters.transfers_executed;
        }
    });
}

int gvxc_pipeline_stream(gvxc_pipeline p, const uint8_t* const* frames, int n, int pinned,
                         void (*on_result)(const void* view, size_t bytes, void* user), void* user,
                         long long counters[4]) {
    return guarded([&] {
        gvxc_graph g = p->g;
        if (g->cfg == 4) throw gvx::Error(gvx::ErrorCode::UnknownObject, "config 4 has no image output");
        const std::size_t px = static_cast<std::size_t>(g->width) * static_cast<std::size_t>(g->height);
        const std::size_t out_bytes = (g->cfg == 1 || g->cfg == 5 ? 2u : 1u) * px;
        const gvx::ObjectId in_id = g->cg.input, out_id = g->cg.outputs.at(0);
        long long acc[4] = {0, 0, 0, 0};
        auto take = [&] {
            const void* view = nullptr;
            const gvx::ExecutionReport r = p->p->next_view(out_id, &view);
            if (on_result) on_result(view, out_bytes, user); // before the next submit reuses the staging
            acc[0] += r.counters.kernel_launches;
            acc[1] += r.counters.pixels_read;
            acc[2] += r.counters.pixels_written;
            acc[3] += r.counters.transfers_executed;
        };
        try {
            for (int i = 0; i < n; ++i) {
                if (p->p->pending() >= p->depth) take();
                if (pinned) p->p->submit_pinned(in_id, frames[i], px);
                else p->p->submit(in_id, frames[i], px);
            }
            while (p->p->pending() > 0) take();
        } catch (...) {
            // no DMA may still read the caller's (possibly page-locked) frames
            // after we return, and no stale result may reach the next call
            while (p->p->pending() > 0) {
                try {
                    p->p->next();
                } catch (...) {
                }
            }
            throw;
        }
        if (counters)
            for (int k = 0; k < 4; ++k) counters[k] = acc[k];
    });
}

int gvxc_pipeline_next(gvxc_pipeline p, void* out, long long* hist, double* stats, long long counters[4]) {
    return guarded([&] {
        gvxc_graph g = p->g;
        gvx::ExecutionReport r;
        if (g->cfg != 4 && out) {
            const gvx::ObjectId id = g->cg.outputs.at(0);
            const std::size_t bpp = g->cfg == 1 || g->cfg == 5 ? 2 : 1;
            r = p->p->next_into(id, out, bpp * static_cast<std::size_t>(g->width) * static_cast<std::size_t>(g->height));
        } else {
            r = p->p->next();
            copy_outputs(g, r.outputs, out, hist, stats);
        }
        if (counters) {
            counters[0] = r.counters.kernel_launches;
            counters[1] = r.counters.pixels_read;
            counters[2] = r.counters.pixels_written;
            counters[3] = r.counters.transfers_executed;
        }
    });
}

} // extern "C"

// ------------------------------------------------------------ row bands

struct gvxc_band_s {
    gvxc_graph g = nullptr;
    std::unique_ptr<gvx::BandedSession> own;
    gvx::BandedSession* s = nullptr;
};

struct gvxc_group_s {
    gvxc_graph g = nullptr;
    std::unique_ptr<gvx::BandGroup> group;
    std::vector<std::unique_ptr<gvxc_band_s>> bands;
};

namespace {
gvx::ObjectId band_slot(gvxc_graph g, int slot) {
    if (slot == 0) return g->cg.input;
    if (slot < 1 || slot > static_cast<int>(g->cg.outputs.size()))
        throw gvx::Error(gvx::ErrorCode::UnknownObject, "bad slot");
    return g->cg.outputs[static_cast<std::size_t>(slot - 1)];
}
} // namespace

extern "C" {

int gvxc_band_create(gvxc_graph g, int rank, int world, void* comm, int device, int frames, gvxc_band* out) {
    return guarded([&] {
        auto b = std::make_unique<gvxc_band_s>();
        b->g = g;
        b->own = std::make_unique<gvx::BandedSession>(g->plan, rank, world, comm, device, frames);
        b->s = b->own.get();
        *out = b.release();
    });
}

int gvxc_band_destroy(gvxc_band b) {
    if (b && b->own) delete b; // group members belong to their group
    return 0;
}

int gvxc_band_layout(gvxc_band b, int32_t out[9]) {
    return guarded([&] {
        const gvx::BandLayout l = b->s->layout();
        const int32_t v[9] = {l.rank, l.world, l.width, l.height, l.row0, l.row1, l.src_row0, l.src_row1, l.halo};
        std::memcpy(out, v, sizeof(v));
    });
}

int gvxc_band_tensor(gvxc_band b, int slot, void** dptr, int64_t* pitch, int64_t* fstride, int32_t* first_row,
                     int32_t* rows) {
    return guarded([&] {
        int r0 = 0, n = 0;
        const gvx::DeviceTensor t = b->s->tensor(band_slot(b->g, slot), &r0, &n);
        *dptr = t.data;
        if (pitch) *pitch = t.pitch;
        if (fstride) *fstride = t.frame_stride;
        if (first_row) *first_row = r0;
        if (rows) *rows = n;
    });
}

int gvxc_band_upload(gvxc_band b, int slot, const void* host, size_t pitch, int first_row, int rows, int frame) {
    return guarded([&] { b->s->upload_rows(band_slot(b->g, slot), host, pitch, first_row, rows, frame); });
}

int gvxc_band_download(gvxc_band b, int slot, void* host, size_t pitch, int first_row, int rows, int frame) {
    return guarded([&] { b->s->download_rows(band_slot(b->g, slot), host, pitch, first_row, rows, frame); });
}

int gvxc_band_set_overlap(gvxc_band b, int mode) {
    return guarded([&] { b->s->set_overlap(mode); });
}

int gvxc_band_bind(gvxc_band b, int slot, void* dptr, int64_t pitch, int64_t fstride) {
    return guarded([&] { b->s->bind(band_slot(b->g, slot), gvx::DeviceTensor{dptr, pitch, fstride}); });
}

int gvxc_band_set_stream(gvxc_band b, void* stream) {
    return guarded([&] { b->s->set_stream(stream); });
}

int gvxc_band_launch(gvxc_band b) {
    return guarded([&] { b->s->launch(); });
}

int gvxc_band_sync(gvxc_band b) {
    return guarded([&] { b->s->synchronize(); });
}

int gvxc_band_launches(gvxc_band b) { return b->s->launches_per_run(); }

int gvxc_band_run_host(gvxc_band b, const void* src, size_t src_pitch, int slot, void* dst, size_t dst_pitch,
                       int piece_rows) {
    return guarded([&] { b->s->run_host(src, src_pitch, band_slot(b->g, slot), dst, dst_pitch, piece_rows); });
}

int gvxc_band_describe(gvxc_band b, char* buf, size_t cap) {
    return guarded([&] {
        const std::string d = b->s->describe();
        if (cap) {
            std::strncpy(buf, d.c_str(), cap - 1);
            buf[cap - 1] = '\0';
        }
    });
}

int gvxc_group_create(gvxc_graph g, int n, const int* devices, int frames, gvxc_group* out) {
    return guarded([&] {
        auto gr = std::make_unique<gvxc_group_s>();
        gr->g = g;
        gr->group = std::make_unique<gvx::BandGroup>(g->plan, std::vector<int>(devices, devices + n), frames);
        for (int i = 0; i < n; ++i) {
            auto b = std::make_unique<gvxc_band_s>();
            b->g = g;
            b->s = &gr->group->band(i);
            gr->bands.push_back(std::move(b));
        }
        *out = gr.release();
    });
}

int gvxc_group_destroy(gvxc_group gr) {
    delete gr;
    return 0;
}

int gvxc_group_band(gvxc_group gr, int i, gvxc_band* out) {
    return guarded([&] {
        if (i < 0 || i >= static_cast<int>(gr->bands.size())) throw gvx::Error(gvx::ErrorCode::UnknownObject, "bad band");
        *out = gr->bands[static_cast<std::size_t>(i)].get();
    });
}

int gvxc_group_launch(gvxc_group gr) {
    return guarded([&] { gr->group->launch(); });
}

int gvxc_group_sync(gvxc_group gr) {
    return guarded([&] { gr->group->synchronize(); });
}

} // extern "C"

// ------------------------------------------------------------ graph files

struct gvxc_json_s {
    std::unique_ptr<gvx_json_runner::Loaded> L;
};

extern "C" {

int gvxc_json_roundtrip(const char* text, char* out, size_t cap, size_t* len) {
    return guarded([&] {
        const std::string t = gvx::save_graph_json(gvx::load_graph_json(text));
        if (len) *len = t.size() + 1;
        if (out && cap > 0) {
            const size_t n = std::min(cap - 1, t.size());
            std::memcpy(out, t.data(), n);
            out[n] = 0;
        }
    });
}

int gvxc_json_load(const char* text, gvxc_json* out) {
    return guarded([&] {
        auto g = std::make_unique<gvxc_json_s>();
        g->L = gvx_json_runner::load(text);
        *out = g.release();
    });
}

int gvxc_json_destroy(gvxc_json g) {
    delete g;
    return 0;
}

int gvxc_json_run(gvxc_json g, int naive, unsigned long long seed, uint8_t* out, size_t cap, size_t* len,
                  long long counters[4]) {
    return guarded([&] {
        const std::vector<std::uint8_t> r = gvx_json_runner::run(*g->L, naive != 0, seed);
        if (len) *len = r.size();
        if (out) std::memcpy(out, r.data(), std::min(cap, r.size()));
        if (counters) {
            counters[0] = g->L->counters.kernel_launches;
            counters[1] = g->L->counters.pixels_read;
            counters[2] = g->L->counters.pixels_written;
            counters[3] = g->L->counters.transfers_executed;
        }
    });
}

int gvxc_json_describe(gvxc_json g, int naive, char* buf, size_t cap) {
    return guarded([&] {
        std::string d = naive ? gvx::DeviceSession(g->L->impl).describe() : gvx::DeviceSession(*g->L->plan).describe();
        if (cap) {
            std::strncpy(buf, d.c_str(), cap - 1);
            buf[cap - 1] = '\0';
        }
    });
}

int gvxc_json_bench(gvxc_json g, int naive, int frames, int iters, unsigned long long seed, double out[4]) {
    return guarded([&] {
        const gvx::AppGraph& app = *g->L->lg.graph;
        const gvx::Context& ctx = *g->L->lg.ctx;
        gvx::DeviceSession s = naive ? gvx::DeviceSession(g->L->impl, frames) : gvx::DeviceSession(*g->L->plan, frames);
        double bytes = 0; // algorithmic HBM bytes per execution: source images in, observable images out
        for (gvx::ObjectId id : app.data()) {
            const gvx::DataObject* o = ctx.find(id);
            if (!o || o->is_virtual || o->kind != gvx::ObjKind::Image) continue;
            const gvx::ResolvedDesc d = o->desc();
            const double b = static_cast<double>(d.width) * d.height * gvx::bytes_per_pixel(d.format) * frames;
            if (app.producer(id) == gvx::kInvalidId) {
                if (app.consumers(id).empty()) continue;
                gvx::Buffer in = gvx::random_buffer(d, seed + static_cast<std::uint64_t>(id));
                for (int f = 0; f < frames; ++f) s.upload(id, in, f);
            }
            bytes += b;
        }
        for (int i = 0; i < 3; ++i) s.launch();
        s.synchronize();
        void* ev[2];
        gvxb_event_create(&ev[0]);
        gvxb_event_create(&ev[1]);
        gvxb_ctx c = nullptr;
        gvxb_ctx_create(gvxb_ctx_device(gvx::dev::context()), &c);
        s.set_stream(gvxb_ctx_stream(c));
        s.launch();
        gvxb_event_record(c, ev[0]);
        const long long l0 = gvxb_total_launch_count();
        for (int i = 0; i < iters; ++i) s.launch();
        gvxb_event_record(c, ev[1]);
        s.synchronize();
        float ms = 0;
        gvxb_event_elapsed_ms(ev[0], ev[1], &ms);
        out[0] = ms / iters;
        out[1] = bytes;
        out[2] = static_cast<double>(gvxb_total_launch_count() - l0) / iters;
        out[3] = frames;
        s.set_stream(nullptr);
        gvxb_event_destroy(ev[0]);
        gvxb_event_destroy(ev[1]);
        gvxb_ctx_destroy(c);
    });
}

int gvxc_json_pass_stats(gvxc_json g, long long st[8]) {
    const gvx::PassStats& p = g->L->plan->stats;
    const long long v[8] = {p.nodes_before, p.nodes_alive, p.nodes_removed, p.transfers_naive,
                            p.transfers_optimized, p.fused_groups, p.launches_before, p.launches_after};
    std::memcpy(st, v, sizeof(v));
    return 0;
}

} // extern "C"
