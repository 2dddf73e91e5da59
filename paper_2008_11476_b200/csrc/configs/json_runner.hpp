// Header-only driver for graph-description files, compiled against BOTH the
// product API and the reference (oracle/ref_shim.cpp, -Dgvx=gvxref) so that
// the two sides load, verify, expand and execute a graph file the same way:
//   load_graph_json -> verify -> expand -> verify -> run_plan | run_naive
// with reference random_buffer inputs (seed + object id) for every
// non-virtual source image, and the declared outputs serialised as
//   [u32 kind][u32 nbytes][payload] ...
// kind 0 image (packed bytes), 1 scalar ({u8 real, i64/f64 bits}),
// 2 array (Value slots {u8 real, 8 bytes} x n), 3 distribution (i64 counts).
#pragma once

#include "graphvx/execute.hpp"
#include "graphvx/graph_io.hpp"
#include "graphvx/optimize.hpp"
#include "graphvx/registry.hpp"
#include "graphvx/verify.hpp"

#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

// the reference-side build renames this namespace (its inline functions
// would otherwise share mangled names with the product's copies)
#ifndef GVX_JSON_RUNNER_NS
#define GVX_JSON_RUNNER_NS gvx_json_runner
#endif

namespace GVX_JSON_RUNNER_NS {

struct Loaded {
    gvx::LoadedGraph lg;
    gvx::VerifiedGraph impl;
    std::unique_ptr<gvx::OptimizedPlan> plan;
    gvx::ExecCounters counters;
};

inline std::string first_diag(const gvx::VerifyResult& r) {
    return r.diagnostics.empty() ? std::string("?") : r.diagnostics.front().render();
}

inline std::unique_ptr<Loaded> load(const std::string& text) {
    auto L = std::make_unique<Loaded>();
    L->lg = gvx::load_graph_json(text);
    gvx::VerifyResult vr = gvx::verify(*L->lg.graph);
    if (!vr.ok()) throw std::runtime_error("verify: " + first_diag(vr));
    gvx::AppGraph& impl = gvx::expand(vr.verified, *L->lg.ctx);
    gvx::VerifyResult ir = gvx::verify(impl);
    if (!ir.ok()) throw std::runtime_error("verify(impl): " + first_diag(ir));
    L->impl = ir.verified;
    L->plan = std::make_unique<gvx::OptimizedPlan>(gvx::optimize(L->impl, *L->lg.ctx));
    return L;
}

inline void put_u32(std::vector<std::uint8_t>& out, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}

inline void put_value(std::vector<std::uint8_t>& out, const gvx::Value& v) {
    out.push_back(v.real ? 1 : 0);
    std::uint8_t b[8];
    if (v.real) std::memcpy(b, &v.f, 8);
    else std::memcpy(b, &v.i, 8);
    out.insert(out.end(), b, b + 8);
}

/// Executes the loaded graph; returns the serialised declared outputs.
inline std::vector<std::uint8_t> run(Loaded& L, bool naive, std::uint64_t seed) {
    const gvx::AppGraph& app = *L.lg.graph;
    gvx::InputMap inputs;
    for (gvx::ObjectId id : app.data()) {
        const gvx::DataObject* o = L.lg.ctx->find(id);
        if (!o || o->is_virtual || o->kind != gvx::ObjKind::Image) continue;
        if (app.producer(id) != gvx::kInvalidId || app.consumers(id).empty()) continue;
        gvx::Buffer b = gvx::random_buffer(o->desc(), seed + static_cast<std::uint64_t>(id));
        b.id = id;
        inputs[id] = std::move(b);
    }
    gvx::ExecutionReport rep = naive ? gvx::run_naive(L.impl, inputs) : gvx::run_plan(*L.plan, inputs);
    L.counters = rep.counters;
    std::vector<std::uint8_t> out;
    for (gvx::ObjectId id : L.lg.declared_outputs) {
        auto it = rep.outputs.find(id);
        if (it == rep.outputs.end()) throw std::runtime_error("declared output missing from the report");
        const gvx::Buffer& b = it->second;
        std::vector<std::uint8_t> payload;
        std::uint32_t kind = 0;
        if (b.desc.kind == gvx::ObjKind::Image) {
            payload = b.bytes;
        } else if (b.desc.kind == gvx::ObjKind::Scalar) {
            kind = 1;
            put_value(payload, b.scalar);
        } else if (b.has_dist) {
            kind = 3;
            for (std::int64_t c : b.dist.counts) {
                std::uint8_t x[8];
                std::memcpy(x, &c, 8);
                payload.insert(payload.end(), x, x + 8);
            }
        } else {
            kind = 2;
            for (const gvx::Value& v : b.elements) put_value(payload, v);
        }
        put_u32(out, kind);
        put_u32(out, static_cast<std::uint32_t>(payload.size()));
        out.insert(out.end(), payload.begin(), payload.end());
    }
    return out;
}

} // namespace GVX_JSON_RUNNER_NS
