// ORACLE (test infrastructure only — never linked into the product).
//
// C entry points over the UNMODIFIED reference library, compiled from
// /root/reference/proj/src with -Dgvx=gvxref by oracle/Makefile into
// oracle/_ref/liboracle_ref.so.  Used by tests/ (parity), bench.py
// (--impl reference and the cpu_baseline leg) and nothing else.
//
// The config graphs come from the same builder the product uses
// (paper_2008_11476_b200/csrc/configs/config_graphs.hpp) compiled here
// against the reference headers, with NON-virtual intermediates because the
// reference's expand() rejects virtual images (SURVEY.md §0 finding 1;
// run_naive results are identical either way).
#include "graphvx/execute.hpp"
#include "graphvx/optimize.hpp"
#include "graphvx/registry.hpp"
#include "graphvx/verify.hpp"

#include "../paper_2008_11476_b200/csrc/configs/config_graphs.hpp"
#ifdef OREF_GRAPH_IO
#define GVX_JSON_RUNNER_NS gvxref_json_runner
#include "../paper_2008_11476_b200/csrc/configs/json_runner.hpp"
#endif

#include <chrono>
#include <cstring>
#include <string>

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* oref_last_error(void) { return g_err.c_str(); }

/// The reference's random_buffer bytes (ref:src/execute.cpp:125-167).
int oref_random_image(int w, int h, int fmt, unsigned long long seed, unsigned char* out) {
    try {
        gvx::ResolvedDesc d;
        d.kind = gvx::ObjKind::Image;
        d.width = w;
        d.height = h;
        d.format = static_cast<gvx::ImageFormat>(fmt);
        gvx::Buffer b = gvx::random_buffer(d, seed);
        std::memcpy(out, b.bytes.data(), b.bytes.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

/// Runs config `cfg` through verify -> expand -> verify -> run_naive on the
/// reference CPU engine.  Outputs: cfg1/5 S16 magnitude, cfg2 U8 mask,
/// cfg3 U8 image into `out`; cfg4 histogram (256 int64) into `hist` and
/// {mean, stddev} into `stats`.  `seconds` gets the run_naive wall time.
int oref_run_config(int cfg, int w, int h, const unsigned char* in, void* out, long long* hist, double* stats,
                    double* seconds) {
    try {
        gvx::Context ctx;
        gvx_configs::ConfigGraph cg = gvx_configs::build_config(ctx, cfg, w, h, /*virtual_mid=*/false);
        gvx::VerifiedGraph impl = gvx_configs::verified_impl(ctx, *cg.graph);
        gvx::ResolvedDesc d;
        d.kind = gvx::ObjKind::Image;
        d.width = w;
        d.height = h;
        d.format = gvx::ImageFormat::U8;
        gvx::Buffer src = gvx::Buffer::image(d);
        std::memcpy(src.bytes.data(), in, static_cast<std::size_t>(w) * h);
        gvx::InputMap inputs;
        inputs[cg.input] = src;
        auto t0 = std::chrono::steady_clock::now();
        gvx::ExecutionReport r = gvx::run_naive(impl, inputs);
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (cfg == 4) {
            const gvx::Buffer& hb = r.outputs.at(cg.outputs[0]);
            for (std::size_t i = 0; i < hb.dist.counts.size() && hist; ++i) hist[i] = hb.dist.counts[i];
            if (stats) {
                stats[0] = r.outputs.at(cg.outputs[1]).scalar.as_real();
                stats[1] = r.outputs.at(cg.outputs[2]).scalar.as_real();
            }
        } else if (out) {
            const gvx::Buffer& ob = r.outputs.at(cg.outputs[0]);
            std::memcpy(out, ob.bytes.data(), ob.bytes.size());
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

/// Reference event counters of run_naive for config `cfg` (launches,
/// pixels read, pixels written, transfers).
int oref_config_counters(int cfg, int w, int h, const unsigned char* in, long long* counters) {
    try {
        gvx::Context ctx;
        gvx_configs::ConfigGraph cg = gvx_configs::build_config(ctx, cfg, w, h, false);
        gvx::VerifiedGraph impl = gvx_configs::verified_impl(ctx, *cg.graph);
        gvx::ResolvedDesc d;
        d.kind = gvx::ObjKind::Image;
        d.width = w;
        d.height = h;
        d.format = gvx::ImageFormat::U8;
        gvx::Buffer src = gvx::Buffer::image(d);
        std::memcpy(src.bytes.data(), in, static_cast<std::size_t>(w) * h);
        gvx::InputMap inputs;
        inputs[cg.input] = src;
        gvx::ExecutionReport r = gvx::run_naive(impl, inputs);
        counters[0] = r.counters.kernel_launches;
        counters[1] = r.counters.pixels_read;
        counters[2] = r.counters.pixels_written;
        counters[3] = r.counters.transfers_executed;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

#ifdef OREF_GRAPH_IO
/// save_graph_json(load_graph_json(text)) of the reference.
int oref_json_roundtrip(const char* text, char* out, size_t cap, size_t* len) {
    try {
        const std::string t = gvx::save_graph_json(gvx::load_graph_json(text));
        *len = t.size() + 1;
        if (out && cap > 0) {
            const size_t n = t.size() < cap - 1 ? t.size() : cap - 1;
            std::memcpy(out, t.data(), n);
            out[n] = 0;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

/// The reference pipeline over a graph file (configs/json_runner.hpp),
/// run_naive with random_buffer(seed + id) inputs.
int oref_json_run(const char* text, unsigned long long seed, unsigned char* out, size_t cap, size_t* len,
                  long long* counters) {
    try {
        auto L = gvxref_json_runner::load(text);
        const std::vector<std::uint8_t> r = gvxref_json_runner::run(*L, true, seed);
        *len = r.size();
        if (out) std::memcpy(out, r.data(), r.size() < cap ? r.size() : cap);
        if (counters) {
            counters[0] = L->counters.kernel_launches;
            counters[1] = L->counters.pixels_read;
            counters[2] = L->counters.pixels_written;
            counters[3] = L->counters.transfers_executed;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
int oref_have_graph_io(void) { return 1; }
#else
int oref_have_graph_io(void) { return 0; }
#endif

} // extern "C"
