// vxProcessGraph on the B200: Buffers, device programs, sessions and the
// run_naive / run_plan entry points.
//
// Host contract kept from ref:src/execute.cpp:
//   Buffer layout, load/store, byte_equal     :14-123
//   random_buffer (mt19937_64 streams)        :125-167
//   input binding rules and errors            :300-346
//   outputs = every produced non-virtual obj  :862-876
//   transfers_executed                        :880-897
// Everything per pixel runs on the device through include/gvxb.h.
#include "graphvx/device.hpp"
#include "hostcopy.hpp"
#include "program.hpp"

#include <algorithm>
#include <deque>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <future>
#include <random>
#include <sstream>
#include <unordered_map>

namespace gvx {

// ================================================================== Buffer

namespace {
std::size_t packed_bytes(const ResolvedDesc& d) {
    return static_cast<std::size_t>(d.width) * static_cast<std::size_t>(d.height) *
           static_cast<std::size_t>(bytes_per_pixel(d.format));
}
} // namespace

Buffer Buffer::image(const ResolvedDesc& d) {
    Buffer b;
    b.desc = d;
    b.bytes.assign(packed_bytes(d), 0);
    return b;
}

Buffer Buffer::scalar_value(ScalarType t, Value v) {
    Buffer b;
    b.desc.kind = ObjKind::Scalar;
    b.desc.element_type = t;
    b.scalar = v;
    return b;
}

Value Buffer::load(int x, int y, Channel ch) const {
    const std::size_t i = static_cast<std::size_t>(y) * static_cast<std::size_t>(desc.width) + x;
    const std::uint8_t* p = bytes.data();
    switch (desc.format) {
    case ImageFormat::U8: return Value::of_int(p[i]);
    case ImageFormat::U16: {
        std::uint16_t v;
        std::memcpy(&v, p + 2 * i, 2);
        return Value::of_int(v);
    }
    case ImageFormat::S16: {
        std::int16_t v;
        std::memcpy(&v, p + 2 * i, 2);
        return Value::of_int(v);
    }
    case ImageFormat::S32: {
        std::int32_t v;
        std::memcpy(&v, p + 4 * i, 4);
        return Value::of_int(v);
    }
    case ImageFormat::F32: {
        float v;
        std::memcpy(&v, p + 4 * i, 4);
        return Value::of_real(v);
    }
    case ImageFormat::RGB: return Value::of_int(p[3 * i + (ch == Channel::G ? 1 : ch == Channel::B ? 2 : 0)]);
    case ImageFormat::UYVY: {
        const std::size_t row = static_cast<std::size_t>(y) * desc.width * 2;
        if (ch == Channel::U) return Value::of_int(p[row + 4 * (x / 2)]);
        if (ch == Channel::V) return Value::of_int(p[row + 4 * (x / 2) + 2]);
        return Value::of_int(p[row + 2 * x + 1]);
    }
    case ImageFormat::UNRESOLVED: break;
    }
    throw Error(ErrorCode::BadFormat, "load from unresolved image");
}

void Buffer::store(int x, int y, Channel ch, const Value& v) {
    const std::size_t i = static_cast<std::size_t>(y) * static_cast<std::size_t>(desc.width) + x;
    std::uint8_t* p = bytes.data();
    switch (desc.format) {
    case ImageFormat::U8: p[i] = static_cast<std::uint8_t>(v.i); return;
    case ImageFormat::U16: {
        auto s = static_cast<std::uint16_t>(v.i);
        std::memcpy(p + 2 * i, &s, 2);
        return;
    }
    case ImageFormat::S16: {
        auto s = static_cast<std::int16_t>(v.i);
        std::memcpy(p + 2 * i, &s, 2);
        return;
    }
    case ImageFormat::S32: {
        auto s = static_cast<std::int32_t>(v.i);
        std::memcpy(p + 4 * i, &s, 4);
        return;
    }
    case ImageFormat::F32: {
        auto s = static_cast<float>(v.as_real());
        std::memcpy(p + 4 * i, &s, 4);
        return;
    }
    case ImageFormat::RGB: p[3 * i + (ch == Channel::G ? 1 : ch == Channel::B ? 2 : 0)] = static_cast<std::uint8_t>(v.i); return;
    default: break;
    }
    throw Error(ErrorCode::BadFormat, "store into unsupported format");
}

bool Buffer::byte_equal(const Buffer& o) const {
    if (desc.kind != o.desc.kind) return false;
    switch (desc.kind) {
    case ObjKind::Image: return bytes == o.bytes;
    case ObjKind::Scalar: return scalar == o.scalar;
    case ObjKind::Array:
        if (has_dist != o.has_dist) return false;
        return has_dist ? dist.counts == o.dist.counts : elements == o.elements;
    case ObjKind::Matrix: return elements == o.elements;
    }
    return false;
}

Buffer random_buffer(const ResolvedDesc& desc, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    Buffer b;
    b.desc = desc;
    if (desc.kind == ObjKind::Image) {
        b = Buffer::image(desc);
        const std::size_t n = b.bytes.size();
        std::uint8_t* p = b.bytes.data();
        switch (desc.format) {
        case ImageFormat::F32: {
            std::uniform_real_distribution<float> d(0.0f, 255.0f);
            for (std::size_t i = 0; i < n / 4; ++i) {
                float v = d(rng);
                std::memcpy(p + 4 * i, &v, 4);
            }
            break;
        }
        case ImageFormat::S16: {
            std::uniform_int_distribution<int> d(-32768, 32767);
            for (std::size_t i = 0; i < n / 2; ++i) {
                auto v = static_cast<std::int16_t>(d(rng));
                std::memcpy(p + 2 * i, &v, 2);
            }
            break;
        }
        case ImageFormat::U16: {
            std::uniform_int_distribution<int> d(0, 65535);
            for (std::size_t i = 0; i < n / 2; ++i) {
                auto v = static_cast<std::uint16_t>(d(rng));
                std::memcpy(p + 2 * i, &v, 2);
            }
            break;
        }
        case ImageFormat::S32: {
            std::uniform_int_distribution<std::int32_t> d(-100000, 100000);
            for (std::size_t i = 0; i < n / 4; ++i) {
                std::int32_t v = d(rng);
                std::memcpy(p + 4 * i, &v, 4);
            }
            break;
        }
        default: {
            std::uniform_int_distribution<int> d(0, 255);
            for (std::size_t i = 0; i < n; ++i) p[i] = static_cast<std::uint8_t>(d(rng));
            break;
        }
        }
        return b;
    }
    if (desc.kind == ObjKind::Scalar) {
        std::uniform_int_distribution<int> d(0, 255);
        const int v = d(rng);
        b.scalar = is_float(desc.element_type) ? Value::of_real(static_cast<double>(v)) : Value::of_int(v);
        return b;
    }
    std::uniform_int_distribution<int> d(-8, 8);
    const std::int64_t n = desc.kind == ObjKind::Array ? desc.capacity
                                                       : static_cast<std::int64_t>(desc.rows) * desc.cols;
    for (std::int64_t i = 0; i < n; ++i) {
        const int v = d(rng);
        b.elements.push_back(is_float(desc.element_type) ? Value::of_real(v) : Value::of_int(v));
    }
    return b;
}

// ============================================================ device layer

namespace dev {

void check(int status, const char* what) {
    if (status == GVXB_OK) return;
    const std::string msg = std::string(what) + ": " + gvxb_last_error();
    if (status >= 1 && status <= 20) throw Error(static_cast<ErrorCode>(status - 1), msg);
    if (status == GVXB_ERR_INVALID) throw Error(ErrorCode::BadKernel, msg);
    throw Error(ErrorCode::UnsupportedKind, msg);
}

gvxb_ctx context() {
    static std::mutex m;
    static gvxb_ctx ctx = nullptr;
    std::lock_guard<std::mutex> lock(m);
    if (ctx) return ctx;
    int n = 0;
    if (gvxb_device_count(&n) != GVXB_OK || n == 0)
        throw Error(ErrorCode::UnsupportedKind,
                    "no CUDA device: graphvx-b200 executes graphs only on the GPU (no host fallback)");
    int dev = 0;
    if (const char* e = std::getenv("GVX_DEVICE")) dev = std::atoi(e);
    check(gvxb_ctx_create(dev, &ctx), "gvxb_ctx_create");
    return ctx;
}

long long launch_count() {
    context();
    return gvxb_total_launch_count();
}

/// A context of its own (stream, status word, read counter) on the library's
/// device: sessions executing concurrently never share error flags or
/// counters (the reference allows concurrent run_* calls).
gvxb_ctx own_context(int device) {
    gvxb_ctx c = nullptr;
    check(gvxb_ctx_create(device >= 0 ? device : gvxb_ctx_device(context()), &c), "gvxb_ctx_create");
    return c;
}

namespace {

// ------------------------------------------------------------ JIT modules

std::mutex g_module_mu;
// process-lifetime caches are intentionally leaked: tearing down device
// objects from static destructors races the CUDA runtime's own teardown
std::unordered_map<std::string, gvxb_module>& module_cache() {
    static auto* cache = new std::unordered_map<std::string, gvxb_module>();
    return *cache;
}

gvxb_module compile(const jit::NodeProgram& prog) {
    const std::string& src = prog.kernels.at(0).source;
    std::string key = src;
    for (const auto& k : prog.kernels) key += "|" + k.name;
    {
        std::lock_guard<std::mutex> lock(g_module_mu);
        auto it = module_cache().find(key);
        if (it != module_cache().end()) return it->second;
    }
    if (const char* dir = std::getenv("GVX_DUMP_JIT")) { // debugging aid: keep the generated CUDA
        const std::string path = std::string(dir) + "/" + prog.kernels.at(0).name + "_" +
                                 std::to_string(std::hash<std::string>{}(key) % 1000000007ull) + ".cu";
        if (FILE* f = std::fopen(path.c_str(), "w")) {
            std::fwrite(src.data(), 1, src.size(), f);
            std::fclose(f);
        }
    }
    std::vector<const char*> names;
    for (const auto& k : prog.kernels) names.push_back(k.name.c_str());
    gvxb_module m = nullptr;
    const int rc = gvxb_jit_build(context(), src.c_str(), names.data(), static_cast<int>(names.size()), &m);
    if (rc != GVXB_OK)
        throw Error(ErrorCode::UnsupportedKind, std::string("device code generation failed: ") + gvxb_last_error());
    std::lock_guard<std::mutex> lock(g_module_mu);
    auto [it, fresh] = module_cache().emplace(key, m);
    if (!fresh) gvxb_jit_free(m);
    return it->second;
}

jit::SlotInfo slot_of(const VerifiedGraph& vg, ObjectId id) {
    jit::SlotInfo s;
    if (id == kInvalidId) return s;
    s.desc = vg.desc(id);
    switch (s.desc.kind) {
    case ObjKind::Image: s.kind = jit::SlotKind::Image; break;
    case ObjKind::Scalar: s.kind = jit::SlotKind::Scalar; break;
    case ObjKind::Array: s.kind = jit::SlotKind::Array; break;
    case ObjKind::Matrix: s.kind = jit::SlotKind::Matrix; break;
    }
    return s;
}

std::vector<Value> matrix_for(const Unit& u, const Context& ctx,
                              const std::map<ObjectId, std::vector<Value>>& matrices) {
    for (ObjectId id : u.in_ids) {
        if (id == kInvalidId) continue;
        const DataObject* o = ctx.find(id);
        if (!o || o->kind != ObjKind::Matrix) continue;
        auto it = matrices.find(id);
        return it != matrices.end() ? it->second : o->matrix_values;
    }
    return {};
}

Unit jit_unit(const OperatorNode& n, const VerifiedGraph& vg,
              const std::map<ObjectId, std::vector<Value>>& matrices) {
    if (!n.abstraction)
        throw Error(ErrorCode::UnknownKernel, "node '" + n.kernel + "' has no abstraction kernel (expand first)");
    Unit u;
    u.kind = Unit::Kind::Jit;
    u.k = n.abstraction;
    u.label = n.label.empty() ? n.kernel : n.label;
    u.covers = {n.id};
    const auto& ps = u.k->signature.params;
    for (std::size_t i = 0; i < ps.size(); ++i) {
        const Binding* b = n.binding_for(static_cast<int>(i));
        const ObjectId id = b ? b->object : kInvalidId;
        if (ps[i].direction == Direction::Input) {
            u.in_ids.push_back(id);
            u.in_slots.push_back(slot_of(vg, id));
            if (id != kInvalidId) u.reads.push_back(id);
        } else {
            u.out_ids.push_back(id);
            u.out_slots.push_back(slot_of(vg, id));
            if (id != kInvalidId) u.writes.push_back(id);
        }
    }
    std::int64_t r = 0, w = 0;
    const bool stat = static_counts(n, vg, r, w);
    u.prog = jit::lower_node(*u.k, u.in_slots, u.out_slots, matrix_for(u, vg.context(), matrices), !stat);
    const ResolvedDesc* d = nullptr;
    if (u.prog.dims_from >= 0 && u.prog.dims_from < static_cast<int>(u.in_slots.size()))
        d = &u.in_slots[static_cast<std::size_t>(u.prog.dims_from)].desc;
    else if (!u.out_slots.empty() && u.out_slots[0].kind != jit::SlotKind::None)
        d = &u.out_slots[0].desc;
    if (d) {
        u.width = d->width;
        u.height = d->height;
    }
    u.static_writes = w;
    u.device_counts_reads = u.prog.counts_reads;
    u.static_reads = u.prog.counts_reads ? 0 : r;
    return u;
}

/// Generic fused regions (jit::lower_region): maximal convex DAG regions of
/// the remaining executed point / local nodes over images of one size, each
/// one kernel with its intermediates in shared memory.  Returns the units
/// and the executed nodes they cover; a region that cannot be lowered
/// (run-time typed bodies, shared memory) falls back to per-node kernels.
std::vector<Unit> region_units(const AppGraph& fg, const VerifiedGraph& fused, const std::set<ObjectId>& taken,
                               const std::map<ObjectId, std::vector<Value>>& matrices,
                               const std::map<ObjectId, std::pair<long long, long long>>& known, std::set<ObjectId>& covered) {
    std::vector<Unit> units;
    if (std::getenv("GVX_NO_REGIONS")) return units;
    const Context& ctx = fused.context();
    std::map<ObjectId, std::vector<ObjectId>> readers;
    std::map<ObjectId, ObjectId> writer;
    for (const OperatorNode& n : fg.nodes())
        for (const Binding& b : n.bindings) {
            if (b.direction == Direction::Input) readers[b.object].push_back(n.id);
            else writer[b.object] = n.id;
        }
    auto img_dims = [&](ObjectId id, int& w, int& h) {
        if (id == kInvalidId) return true;
        const ResolvedDesc& d = fused.desc(id);
        if (d.kind != ObjKind::Image) return true;
        if (w < 0) w = d.width, h = d.height;
        return d.width == w && d.height == h;
    };
    // candidates
    std::map<ObjectId, std::pair<int, int>> dims;
    std::vector<ObjectId> order = fg.topo_sort();
    std::set<ObjectId> cand;
    for (ObjectId nid : order) {
        if (taken.count(nid)) continue;
        const OperatorNode* n = fg.node(nid);
        if (!n || !n->abstraction) continue;
        const AbstractionKind kk = n->abstraction->kind;
        if (kk != AbstractionKind::Point && kk != AbstractionKind::Local) continue;
        if (kk == AbstractionKind::Local && (n->abstraction->local().median3x3 || n->abstraction->local().window_w > 9 ||
                                             n->abstraction->local().window_h > 9))
            continue;
        std::int64_t r = 0, w = 0;
        if (!static_counts(*n, fused, r, w)) continue;
        int W = -1, H = -1;
        bool ok = true;
        for (const Binding& b : n->bindings) {
            ok = ok && img_dims(b.object, W, H);
            if (b.direction == Direction::Output) {
                const ResolvedDesc& d = fused.desc(b.object);
                ok = ok && d.kind == ObjKind::Image &&
                     (d.format == ImageFormat::U8 || d.format == ImageFormat::U16 || d.format == ImageFormat::S16 ||
                      d.format == ImageFormat::S32 || d.format == ImageFormat::F32);
            }
        }
        if (!ok || W < 0) continue;
        cand.insert(nid);
        dims[nid] = {W, H};
    }
    // reachability over the executed graph (small graphs)
    std::map<ObjectId, std::set<ObjectId>> succ;
    for (const OperatorNode& n : fg.nodes())
        for (const Binding& b : n.bindings)
            if (b.direction == Direction::Output)
                for (ObjectId c : readers[b.object]) succ[n.id].insert(c);
    auto reaches = [&](ObjectId from, const std::set<ObjectId>& targets, const std::set<ObjectId>& avoid) {
        std::vector<ObjectId> st{from};
        std::set<ObjectId> seen{from};
        while (!st.empty()) {
            const ObjectId x = st.back();
            st.pop_back();
            for (ObjectId y : succ[x]) {
                if (targets.count(y)) return true;
                if (avoid.count(y) || !seen.insert(y).second) continue;
                st.push_back(y);
            }
        }
        return false;
    };
    auto convex = [&](const std::set<ObjectId>& S) {
        for (const OperatorNode& m : fg.nodes()) {
            if (S.count(m.id)) continue;
            bool from_s = false;
            for (ObjectId x : S) from_s = from_s || succ[x].count(m.id) || reaches(x, {m.id}, S);
            if (from_s && reaches(m.id, S, {})) return false;
        }
        return true;
    };
    // grow regions along candidate producer -> consumer edges, topo order
    std::map<ObjectId, int> region_of;
    std::vector<std::set<ObjectId>> regions;
    for (ObjectId nid : order) {
        if (!cand.count(nid)) continue;
        const OperatorNode* n = fg.node(nid);
        // join every producer region it can (merging them) while the union stays convex
        std::set<ObjectId> S{nid};
        std::set<int> merged;
        for (const Binding& b : n->bindings) {
            if (b.direction != Direction::Input) continue;
            auto w = writer.find(b.object);
            if (w == writer.end() || !region_of.count(w->second)) continue;
            const int r = region_of[w->second];
            if (merged.count(r) || regions[static_cast<std::size_t>(r)].empty()) continue;
            if (dims[*regions[static_cast<std::size_t>(r)].begin()] != dims[nid]) continue;
            std::set<ObjectId> T = S;
            T.insert(regions[static_cast<std::size_t>(r)].begin(), regions[static_cast<std::size_t>(r)].end());
            if (!convex(T)) continue;
            S = std::move(T);
            merged.insert(r);
        }
        for (int r : merged) regions[static_cast<std::size_t>(r)].clear();
        regions.push_back(S);
        for (ObjectId m : S) region_of[m] = static_cast<int>(regions.size()) - 1;
    }
    for (const std::set<ObjectId>& S : regions) {
        // merged-away (empty) regions and single point nodes run as per-node
        // kernels; a single local node takes the region code too (vector
        // staging and stores, separable box sums: laplacian.json 584 -> 647
        // Gpx/s); GVX_REGION_NOSINGLE=1 keeps it a per-node kernel
        static const bool single = std::getenv("GVX_REGION_NOSINGLE") == nullptr;
        if (S.empty() || (S.size() < 2 && !(single && fg.node(*S.begin())->abstraction->kind == AbstractionKind::Local)))
            continue;
        // members in topological order
        std::vector<const OperatorNode*> mem;
        for (ObjectId nid : order)
            if (S.count(nid)) mem.push_back(fg.node(nid));
        // region objects: images produced by members, and the single-channel
        // images they read from outside (staged into shared memory); halos backwards
        std::map<ObjectId, int> obj_index;
        std::vector<jit::RegionObject> objs;
        std::vector<ObjectId> obj_ids;
        std::set<ObjectId> produced;
        for (const OperatorNode* n : mem)
            for (const Binding& b : n->bindings)
                if (b.direction == Direction::Output) produced.insert(b.object);
        auto staged_format = [](ImageFormat f) {
            return f == ImageFormat::U8 || f == ImageFormat::U16 || f == ImageFormat::S16 || f == ImageFormat::S32 ||
                   f == ImageFormat::F32;
        };
        for (const OperatorNode* n : mem)
            for (const Binding& b : n->bindings) {
                if (obj_index.count(b.object) || b.object == kInvalidId) continue;
                const ResolvedDesc& d = fused.desc(b.object);
                if (d.kind != ObjKind::Image) continue;
                if (b.direction == Direction::Input && !produced.count(b.object) && !staged_format(d.format)) continue;
                obj_index[b.object] = static_cast<int>(objs.size());
                jit::RegionObject ro;
                ro.format = d.format;
                objs.push_back(ro);
                obj_ids.push_back(b.object);
            }
        bool ok = true;
        for (auto it = mem.rbegin(); it != mem.rend(); ++it) {
            const OperatorNode* n = *it;
            int hx = 0, hy = 0; // halo of this node's outputs
            for (const Binding& b : n->bindings)
                if (b.direction == Direction::Output) {
                    hx = std::max(hx, objs[static_cast<std::size_t>(obj_index[b.object])].halo_x);
                    hy = std::max(hy, objs[static_cast<std::size_t>(obj_index[b.object])].halo_y);
                }
            const bool local = n->abstraction->kind == AbstractionKind::Local;
            const int rx = local ? n->abstraction->local().window_w / 2 : 0;
            const int ry = local ? n->abstraction->local().window_h / 2 : 0;
            const auto& ps = n->abstraction->signature.params;
            int slot = 0;
            for (std::size_t i = 0; i < ps.size(); ++i) {
                if (ps[i].direction != Direction::Input) continue;
                const int in_slot = slot++;
                const Binding* b = n->binding_for(static_cast<int>(i));
                if (!b || !obj_index.count(b->object)) continue;
                // the window radius applies to inputs the taps read through a window
                const bool win = local && n->abstraction->local().tap_body &&
                                 jit::reads_window(*n->abstraction->local().tap_body, in_slot);
                jit::RegionObject& ro = objs[static_cast<std::size_t>(obj_index[b->object])];
                ro.halo_x = std::max(ro.halo_x, hx + (win ? rx : 0));
                ro.halo_y = std::max(ro.halo_y, hy + (win ? ry : 0));
            }
        }
        for (const jit::RegionObject& ro : objs) ok = ok && ro.halo_x <= 8 && ro.halo_y <= 8;
        if (!ok) continue;
        Unit u;
        u.kind = Unit::Kind::Jit;
        u.k = mem.back()->abstraction;
        u.label = "region";
        // stored objects: consumed outside the region or observable
        std::vector<jit::SlotInfo> outs;
        for (std::size_t o = 0; o < objs.size(); ++o) {
            const ObjectId id = obj_ids[o];
            if (!produced.count(id)) continue;
            bool outside = false;
            for (ObjectId r : readers[id]) outside = outside || !S.count(r);
            const DataObject* ob = ctx.find(id);
            if (outside || !ob || !ob->is_virtual) {
                objs[o].store = static_cast<int>(outs.size());
                outs.push_back(slot_of(fused, id));
                u.out_ids.push_back(id);
                u.writes.push_back(id);
            }
        }
        std::vector<jit::RegionNode> rnodes;
        std::map<ObjectId, int> param_of;
        std::vector<jit::SlotInfo> ins;
        std::int64_t reads = 0, writes = 0;
        for (const OperatorNode* n : mem) {
            jit::RegionNode rn;
            rn.k = n->abstraction.get();
            const auto& ps = rn.k->signature.params;
            Unit tmp;
            for (std::size_t i = 0; i < ps.size(); ++i) {
                const Binding* b = n->binding_for(static_cast<int>(i));
                const ObjectId id = b ? b->object : kInvalidId;
                if (ps[i].direction == Direction::Input) {
                    rn.in_slots.push_back(slot_of(fused, id));
                    tmp.in_ids.push_back(id);
                    const bool image = id != kInvalidId && fused.desc(id).kind == ObjKind::Image;
                    if (image && obj_index.count(id)) {
                        rn.in_obj.push_back(obj_index[id]);
                        rn.in_param.push_back(-1);
                        if (!produced.count(id) && !param_of.count(id)) { // staged region input
                            param_of[id] = static_cast<int>(ins.size());
                            ins.push_back(slot_of(fused, id));
                            u.in_ids.push_back(id);
                            u.reads.push_back(id);
                            jit::RegionObject& ro = objs[static_cast<std::size_t>(obj_index[id])];
                            ro.load = param_of[id];
                            auto kr = known.find(id);
                            if (kr != known.end()) ro.ranged = true, ro.lo = kr->second.first, ro.hi = kr->second.second;
                        }
                    } else if (image) {
                        if (!param_of.count(id)) {
                            param_of[id] = static_cast<int>(ins.size());
                            ins.push_back(slot_of(fused, id));
                            u.in_ids.push_back(id);
                            u.reads.push_back(id);
                        }
                        rn.in_obj.push_back(-1);
                        rn.in_param.push_back(param_of[id]);
                    } else {
                        rn.in_obj.push_back(-1);
                        rn.in_param.push_back(-1); // matrices are baked in; scalars make the body run-time typed
                    }
                } else {
                    rn.out_obj.push_back(id != kInvalidId && obj_index.count(id) ? obj_index[id] : -1);
                }
            }
            rn.matrix = matrix_for(tmp, ctx, matrices);
            std::int64_t r = 0, w = 0;
            static_counts(*n, fused, r, w);
            reads += r;
            writes += w;
            rnodes.push_back(std::move(rn));
        }
        u.in_slots = ins;
        u.out_slots = outs;
        try {
            u.prog = jit::lower_region(rnodes, objs, ins, outs);
        } catch (const Error& e) {
            if (std::getenv("GVX_TRACE_REGIONS"))
                std::fprintf(stderr, "[gvx region] %zu nodes not fused: %s\n", mem.size(), e.what());
            continue; // run-time typed parts: per-node kernels
        }
        // row-band support: rows beyond its output rows each input is read at
        {
            int hmax = 0;
            for (const jit::RegionObject& ro : objs) hmax = std::max(hmax, ro.halo_y);
            u.prog.in_halo.assign(ins.size(), hmax); // non-staged (multi-channel) inputs: the largest halo
            for (const jit::RegionObject& ro : objs)
                if (ro.load >= 0) u.prog.in_halo[static_cast<std::size_t>(ro.load)] = ro.halo_y;
        }
        u.width = dims[mem.front()->id].first;
        u.height = dims[mem.front()->id].second;
        u.static_reads = reads;
        u.static_writes = writes;
        u.device_counts_reads = false;
        for (const OperatorNode* n : mem) {
            u.covers.push_back(n->id);
            covered.insert(n->id);
        }
        units.push_back(std::move(u));
    }
    return units;
}

void record_objects(Program& p, const VerifiedGraph& vg) {
    const Context& ctx = vg.context();
    for (const Unit& u : p.units) {
        auto touch = [&](ObjectId id, bool produced) {
            if (id == kInvalidId) return;
            ObjInfo& oi = p.objects[id];
            oi.id = id;
            oi.desc = vg.desc(id);
            const DataObject* o = ctx.find(id);
            oi.is_virtual = o && o->is_virtual;
            oi.produced = oi.produced || produced;
            if (oi.desc.kind == ObjKind::Array) oi.length = static_cast<int>(std::max<std::int64_t>(oi.desc.capacity, 0));
            if (oi.desc.kind == ObjKind::Matrix) oi.length = oi.desc.rows * oi.desc.cols;
        };
        for (ObjectId id : u.reads) touch(id, false);
        for (ObjectId id : u.writes) touch(id, true);
    }
    // array roles from producers
    for (const Unit& u : p.units) {
        auto set_role = [&](ObjectId id, ArrayRole role, int len) {
            if (id == kInvalidId) return;
            ObjInfo& oi = p.objects[id];
            oi.role = role;
            oi.length = std::max(oi.length, len);
        };
        if (u.kind == Unit::Kind::Jit) {
            switch (u.k->kind) {
            case AbstractionKind::Histogram: {
                const HistogramKernel& hk = u.k->histogram();
                set_role(u.out_ids[0], ArrayRole::Distribution, hk.bins);
                ObjInfo& oi = p.objects[u.out_ids[0]];
                oi.bins = hk.bins;
                oi.offset = hk.offset;
                oi.range = hk.range;
                break;
            }
            case AbstractionKind::Reduce:
                if (u.out_ids.size() > 1 && u.out_ids[1] != kInvalidId) set_role(u.out_ids[1], ArrayRole::Location, 2);
                break;
            case AbstractionKind::Table: {
                int n = 256;
                if (!u.in_ids.empty() && p.objects.count(u.in_ids[0])) n = std::max(n, p.objects[u.in_ids[0]].length);
                set_role(u.out_ids[0], ArrayRole::Table, n);
                break;
            }
            default: break;
            }
        } else if (u.kind == Unit::Kind::ConvStats && u.out[1] != kInvalidId) {
            set_role(u.out[1], ArrayRole::Distribution, u.bins);
            ObjInfo& oi = p.objects[u.out[1]];
            oi.bins = u.bins;
            oi.offset = u.offset;
            oi.range = u.range;
        }
    }
}

/// Orders units so every object is written before it is read.
void order_units(Program& p) {
    const std::size_t n = p.units.size();
    std::map<ObjectId, std::size_t> writer;
    for (std::size_t i = 0; i < n; ++i)
        for (ObjectId w : p.units[i].writes) writer[w] = i;
    std::vector<std::set<std::size_t>> succ(n);
    std::vector<int> indeg(n, 0);
    for (std::size_t i = 0; i < n; ++i)
        for (ObjectId r : p.units[i].reads) {
            auto it = writer.find(r);
            if (it != writer.end() && it->second != i && succ[it->second].insert(i).second) ++indeg[i];
        }
    std::vector<std::size_t> order;
    std::vector<bool> done(n, false);
    for (std::size_t round = 0; round < n; ++round)
        for (std::size_t i = 0; i < n; ++i) {
            if (done[i] || indeg[i] != 0) continue;
            done[i] = true;
            order.push_back(i);
            for (std::size_t s : succ[i]) --indeg[s];
            break;
        }
    if (order.size() != n) throw Error(ErrorCode::CycleDetected, "device program has a cyclic dependency");
    std::vector<Unit> sorted;
    for (std::size_t i : order) sorted.push_back(std::move(p.units[i]));
    p.units = std::move(sorted);
}

void compile_all(Program& p) {
    std::vector<std::future<gvxb_module>> jobs;
    context();
    for (Unit& u : p.units)
        if (u.kind == Unit::Kind::Jit) jobs.push_back(std::async(std::launch::async, [&u] { return compile(u.prog); }));
    std::size_t j = 0;
    for (Unit& u : p.units)
        if (u.kind == Unit::Kind::Jit) u.module = jobs[j++].get();
}

} // namespace

std::string Program::describe() const {
    std::ostringstream os;
    os << (naive ? "naive" : "plan") << " program, " << units.size() << " units:";
    for (const Unit& u : units) {
        os << "\n  " << u.label << " [";
        switch (u.kind) {
        case Unit::Kind::Jit: os << "nvrtc " << u.prog.kernels.size() << " kernel(s)"; break;
        case Unit::Kind::Edge: os << "sm_100a fused edge" << (u.with_gauss ? " (+gauss)" : ""); break;
        case Unit::Kind::Harris: os << "sm_100a fused harris"; break;
        case Unit::Kind::Stencil: os << "sm_100a fused stencil k=" << u.ksize << " mode=" << u.mode; break;
        case Unit::Kind::ConvStats: os << "sm_100a fused conv+stats k=" << u.ksize; break;
        }
        os << "] covers " << u.covers.size() << " node(s)";
    }
    return os.str();
}

int Program::launches_per_run(int frames) const {
    int n = 0;
    for (const Unit& u : units) {
        if (u.kind == Unit::Kind::Jit) n += static_cast<int>(u.prog.kernels.size());
        // conv+stats: one kernel whose last CTA finalizes (single frames), else
        // scratch clear + kernel (+ MeanStdDev finalize)
        else if (u.kind == Unit::Kind::ConvStats && frames > 1)
            n += (u.out[2] != kInvalidId || u.out[3] != kInvalidId) ? 3 : 2;
        else n += 1;
    }
    return n;
}

std::shared_ptr<Program> build_naive(const VerifiedGraph& vg, const std::map<ObjectId, std::vector<Value>>& matrices) {
    auto p = std::make_shared<Program>();
    p->naive = true;
    const AppGraph& g = vg.graph();
    for (ObjectId nid : g.topo_sort()) p->units.push_back(jit_unit(*g.node(nid), vg, matrices));
    record_objects(*p, vg);
    compile_all(*p);
    return p;
}

std::shared_ptr<Program> build_plan(const OptimizedPlan& plan, const std::map<ObjectId, std::vector<Value>>& matrices) {
    auto p = std::make_shared<Program>();
    const VerifiedGraph& base = plan.base;
    const VerifiedGraph& fused = plan.fused;
    const AppGraph& bg = base.graph();
    const AppGraph& fg = fused.graph();

    GraphView view;
    view.vg = &base;
    view.ctx = &base.context();
    view.matrices = &matrices;
    std::set<ObjectId> alive_nodes;
    for (ObjectId nid : plan.filtered.alive_nodes()) {
        const OperatorNode* n = bg.node(nid);
        if (!n || !n->abstraction) continue;
        view.nodes.push_back(n);
        alive_nodes.insert(nid);
        std::set<ObjectId> seen;
        for (const Binding& b : n->bindings) {
            if (b.direction == Direction::Input) {
                if (seen.insert(b.object).second) view.readers[b.object].push_back(nid);
            } else {
                view.writer[b.object] = nid;
            }
        }
    }
    std::vector<Unit> aot = match_fused_groups(view);

    // base members of every executed (fused-graph) node
    std::map<ObjectId, std::vector<ObjectId>> members;
    for (const FusedKernel& fk : plan.groups) members[fk.fused_node] = fk.members;
    for (const OperatorNode& fnode : fg.nodes()) {
        if (members.count(fnode.id)) continue;
        for (const OperatorNode* bn : view.nodes)
            if (bn->abstraction == fnode.abstraction && bn->bindings.size() == fnode.bindings.size() &&
                std::equal(bn->bindings.begin(), bn->bindings.end(), fnode.bindings.begin(),
                           [](const Binding& a, const Binding& b) {
                               return a.param == b.param && a.object == b.object && a.direction == b.direction;
                           })) {
                members[fnode.id] = {bn->id};
                break;
            }
    }

    // keep only groups that cover whole executed nodes with static counters
    std::set<ObjectId> covered_fused;
    for (bool changed = true; changed;) {
        changed = false;
        covered_fused.clear();
        for (std::size_t gi = 0; gi < aot.size(); ++gi) {
            Unit& u = aot[gi];
            std::set<ObjectId> cov(u.covers.begin(), u.covers.end());
            bool ok = true;
            std::vector<ObjectId> fnodes;
            std::int64_t reads = 0, writes = 0;
            for (const OperatorNode& fnode : fg.nodes()) {
                auto it = members.find(fnode.id);
                if (it == members.end()) continue;
                std::size_t inside = 0;
                for (ObjectId m : it->second) inside += cov.count(m);
                if (inside == 0) continue;
                if (inside != it->second.size()) {
                    ok = false;
                    break;
                }
                std::int64_t r = 0, w = 0;
                if (!static_counts(fnode, fused, r, w)) {
                    ok = false;
                    break;
                }
                reads += r;
                writes += w;
                fnodes.push_back(fnode.id);
            }
            std::size_t member_total = 0;
            for (ObjectId f : fnodes) member_total += members[f].size();
            if (ok && member_total != cov.size()) ok = false; // group must be exactly a union of executed nodes
            if (!ok) {
                aot.erase(aot.begin() + static_cast<std::ptrdiff_t>(gi));
                changed = true;
                break;
            }
            u.static_reads = reads;
            u.static_writes = writes;
            u.covers = fnodes;
            covered_fused.insert(fnodes.begin(), fnodes.end());
        }
    }
    for (Unit& u : aot) p->units.push_back(std::move(u));
    {
        // value ranges of images the hand-written groups produce (Sobel of
        // U8: |g| <= 1020; magnitude <= 1443), narrower than their formats
        std::map<ObjectId, std::pair<long long, long long>> known;
        for (const Unit& u : p->units)
            if (u.kind == Unit::Kind::Edge) {
                for (int i = 0; i < 2; ++i)
                    if (u.out[i] != kInvalidId) known[u.out[i]] = {-1020, 1020};
                if (u.out[2] != kInvalidId) known[u.out[2]] = {0, 1443};
            }
        std::set<ObjectId> rcov;
        for (Unit& u : region_units(fg, fused, covered_fused, matrices, known, rcov)) p->units.push_back(std::move(u));
        covered_fused.insert(rcov.begin(), rcov.end());
    }
    for (ObjectId nid : fg.topo_sort())
        if (!covered_fused.count(nid)) p->units.push_back(jit_unit(*fg.node(nid), fused, matrices));
    order_units(*p);
    record_objects(*p, base);
    compile_all(*p);
    return p;
}

} // namespace dev

// ============================================================== sessions

/// Pinned double-buffered staging for host<->device image copies: the CPU
/// copy of chunk i+1 into pinned memory overlaps the DMA of chunk i, instead
/// of the driver's synchronous pageable path.
struct Staging {
    static constexpr std::size_t kChunk = std::size_t(2) << 20;
    gvxb_ctx ctx = nullptr;
    void* buf[2] = {nullptr, nullptr};
    void* ev[2] = {nullptr, nullptr};
    bool pending[2] = {false, false};

    explicit Staging(gvxb_ctx c) : ctx(c) {
        for (int i = 0; i < 2; ++i) {
            dev::check(gvxb_host_alloc(kChunk, &buf[i]), "pinned staging allocation");
            dev::check(gvxb_event_create(&ev[i]), "staging event");
        }
    }
    ~Staging() {
        for (int i = 0; i < 2; ++i) {
            if (ev[i]) gvxb_event_sync(ev[i]), gvxb_event_destroy(ev[i]);
            if (buf[i]) gvxb_host_free(buf[i]);
        }
    }
    void wait(int k) {
        if (pending[k]) dev::check(gvxb_event_sync(ev[k]), "staging wait");
        pending[k] = false;
    }
    void mark(int k) {
        dev::check(gvxb_event_record(ctx, ev[k]), "staging event");
        pending[k] = true;
    }

    void upload(char* dst, std::size_t pitch, const std::uint8_t* src, std::size_t row, std::size_t rows) {
        const std::size_t per = std::max<std::size_t>(1, kChunk / row);
        int k = 0;
        for (std::size_t r0 = 0; r0 < rows; r0 += per, k ^= 1) {
            const std::size_t n = std::min(per, rows - r0);
            wait(k);
            dev::parallel_copy(buf[k], src + r0 * row, n * row, /*streaming=*/true);
            dev::check(gvxb_upload_2d(ctx, dst + r0 * pitch, pitch, buf[k], row, row, n), "image upload");
            mark(k);
        }
    }

    void download(std::uint8_t* dst, const char* src, std::size_t pitch, std::size_t row, std::size_t rows) {
        const std::size_t per = std::max<std::size_t>(1, kChunk / row);
        const std::size_t chunks = (rows + per - 1) / per;
        auto issue = [&](std::size_t c) {
            const int k = static_cast<int>(c & 1);
            wait(k);
            const std::size_t r0 = c * per, n = std::min(per, rows - r0);
            dev::check(gvxb_download_2d(ctx, buf[k], row, src + r0 * pitch, pitch, row, n), "image download");
            mark(k);
        };
        for (std::size_t c = 0; c < std::min<std::size_t>(2, chunks); ++c) issue(c);
        for (std::size_t c = 0; c < chunks; ++c) {
            const int k = static_cast<int>(c & 1);
            wait(k);
            const std::size_t r0 = c * per, n = std::min(per, rows - r0);
            dev::parallel_copy(dst + r0 * row, buf[k], n * row);
            if (c + 2 < chunks) issue(c + 2);
        }
    }
};

struct DeviceSession::Impl {
    std::shared_ptr<dev::Program> prog;
    std::unique_ptr<Staging> staging; ///< host runs only (run_naive / run_plan)
    /// optional pinned destinations for image outputs (C facade recycling)
    std::map<ObjectId, std::vector<std::uint8_t>>* out_pool = nullptr;
    /// optional: fill this input Buffer from `src` during its upload (C facade)
    const detail::HostFill* fill = nullptr;
    const VerifiedGraph* exec_graph = nullptr; ///< graph whose outputs are reported
    VerifiedGraph exec_copy;
    int frames = 1;
    gvxb_ctx ctx = nullptr;
    void* stream = nullptr;

    struct Store {
        void* ptr = nullptr;
        std::int64_t pitch = 0;
        std::int64_t fstride = 0;
        bool owned = false;
        int length = 0; ///< arrays: live Value slots for bounds checks
    };
    std::map<ObjectId, Store> store;
    std::vector<void*> scratch; ///< per unit (JIT reduce scratch, conv sums)

    bool owns_ctx = false; ///< ctx created for this storage (destroyed with it)
    int last_launches = 0; ///< kernels the last DeviceSession::launch enqueued

    ~Impl() {
        if (!ctx) return;
        gvxb_sync(ctx);
        for (auto& kv : store)
            if (kv.second.owned) gvxb_free(ctx, kv.second.ptr);
        for (void* s : scratch)
            if (s) gvxb_free(ctx, s);
        if (owns_ctx) gvxb_ctx_destroy(ctx);
    }

    static std::int64_t row_pitch(const ResolvedDesc& d) {
        const std::int64_t row = static_cast<std::int64_t>(d.width) * bytes_per_pixel(d.format);
        return std::max<std::int64_t>(128, (row + 127) / 128 * 128);
    }

    Store& ensure(ObjectId id) {
        auto it = store.find(id);
        if (it != store.end()) return it->second;
        const dev::ObjInfo& oi = prog->objects.at(id);
        Store s;
        s.owned = true;
        std::size_t bytes = 0;
        if (oi.desc.kind == ObjKind::Image) {
            s.pitch = row_pitch(oi.desc);
            s.fstride = s.pitch * oi.desc.height;
            bytes = static_cast<std::size_t>(s.fstride) * frames;
        } else {
            const int n = oi.desc.kind == ObjKind::Scalar ? 1 : std::max(oi.length, 1);
            s.length = oi.desc.kind == ObjKind::Scalar ? 1 : oi.length;
            s.fstride = static_cast<std::int64_t>(n) * 16;
            bytes = static_cast<std::size_t>(s.fstride) * frames;
        }
        dev::check(gvxb_alloc(ctx, bytes, &s.ptr), "device allocation");
        dev::check(gvxb_memset(ctx, s.ptr, 0, bytes), "device clear");
        return store.emplace(id, s).first->second;
    }

    gvxb_image image(ObjectId id) {
        gvxb_image im{};
        if (id == kInvalidId) return im;
        Store& s = ensure(id);
        const ResolvedDesc& d = prog->objects.at(id).desc;
        im.data = s.ptr;
        im.pitch = s.pitch;
        im.width = d.width;
        im.height = d.height;
        im.format = static_cast<int32_t>(d.format);
        im.frames = frames;
        im.frame_stride = s.fstride;
        return im;
    }

    gvxb_value* values(ObjectId id) { return id == kInvalidId ? nullptr : static_cast<gvxb_value*>(ensure(id).ptr); }

    void prepare() {
        for (auto& kv : prog->objects) ensure(kv.first);
        scratch.assign(prog->units.size(), nullptr);
        for (std::size_t i = 0; i < prog->units.size(); ++i) {
            const dev::Unit& u = prog->units[i];
            std::size_t bytes = 0;
            if (u.kind == dev::Unit::Kind::Jit) bytes = u.prog.scratch_bytes_per_frame * frames;
            // conv+stats: sum, sumsq and the one-launch accumulators, zero between runs
            if (u.kind == dev::Unit::Kind::ConvStats)
                bytes = (16 + 8 * static_cast<std::size_t>(std::max(u.bins, 1) + 1)) * static_cast<std::size_t>(frames);
            if (bytes) dev::check(gvxb_alloc(ctx, bytes, &scratch[i]), "scratch allocation");
            if (u.kind == dev::Unit::Kind::ConvStats) dev::check(gvxb_memset(ctx, scratch[i], 0, bytes), "scratch clear");
        }
    }

    void launch_unit(std::size_t idx) {
        const dev::Unit& u = prog->units[idx];
        const gvxb_band full{0, 0, 0, 0, 0};
        (void)full;
        switch (u.kind) {
        case dev::Unit::Kind::Jit: launch_jit(u, scratch[idx]); return;
        case dev::Unit::Kind::Edge: {
            gvxb_edge_args a{};
            a.src = image(u.src);
            a.gx = image(u.out[0]);
            a.gy = image(u.out[1]);
            a.mag = image(u.out[2]);
            a.with_gauss = u.with_gauss ? 1 : 0;
            a.band = gvxb_band{0, a.src.height, a.src.height, 0, 0};
            dev::check(gvxb_edge(ctx, &a), "gvxb_edge");
            return;
        }
        case dev::Unit::Kind::Harris: {
            gvxb_harris_args a{};
            a.src = image(u.src);
            a.mask = image(u.out[0]);
            a.response = image(u.out[1]);
            a.k = u.k_param;
            a.threshold = u.threshold;
            a.band = gvxb_band{0, a.src.height, a.src.height, 0, 0};
            dev::check(gvxb_harris(ctx, &a), "gvxb_harris");
            return;
        }
        case dev::Unit::Kind::Stencil: {
            gvxb_stencil_args a{};
            a.src = image(u.src);
            a.dst = image(u.out[0]);
            a.ksize = u.ksize;
            std::memcpy(a.mask, u.mask, sizeof(a.mask));
            a.div_num = 1;
            a.div_den = u.divisor;
            a.mode = u.mode;
            a.band = gvxb_band{0, a.src.height, a.src.height, 0, 0};
            dev::check(gvxb_stencil_point(ctx, &a), "gvxb_stencil_point");
            return;
        }
        case dev::Unit::Kind::ConvStats: {
            gvxb_conv_stats_args a{};
            a.src = image(u.src);
            a.converted = image(u.out[0]);
            a.ksize = u.ksize;
            std::memcpy(a.mask, u.mask, sizeof(a.mask));
            a.scale = u.divisor;
            a.conv_format = u.conv_format;
            a.shift = u.shift;
            a.wrap = u.wrap;
            a.bins = u.bins;
            a.offset = u.offset;
            a.range = u.range;
            a.hist = values(u.out[1]);
            a.sum = static_cast<int64_t*>(scratch[idx]);
            a.sumsq = static_cast<int64_t*>(scratch[idx]) + frames;
            a.work = static_cast<int64_t*>(scratch[idx]) + 2 * frames;
            a.mean = values(u.out[2]);
            a.stddev = values(u.out[3]);
            dev::check(gvxb_conv_stats(ctx, &a), "gvxb_conv_stats");
            return;
        }
        }
    }

    void launch_jit(const dev::Unit& u, void* scr) {
        const jit::NodeProgram& np = u.prog;
        std::vector<std::uint64_t> f(static_cast<std::size_t>(np.fields()), 0);
        unsigned long long* counter = nullptr;
        std::uint32_t* status = nullptr;
        gvxb_counter_ptr(ctx, &counter);
        gvxb_status_ptr(ctx, &status);
        f[0] = reinterpret_cast<std::uint64_t>(status);
        f[1] = reinterpret_cast<std::uint64_t>(counter);
        f[2] = static_cast<std::uint64_t>(u.width);
        f[3] = static_cast<std::uint64_t>(u.height);
        f[4] = static_cast<std::uint64_t>(frames);
        auto put = [&](int slot, ObjectId id) {
            const std::size_t b = static_cast<std::size_t>(5 + 3 * slot);
            if (id == kInvalidId) return;
            Store& s = ensure(id);
            f[b] = reinterpret_cast<std::uint64_t>(s.ptr);
            const dev::ObjInfo& oi = prog->objects.at(id);
            f[b + 1] = oi.desc.kind == ObjKind::Image ? static_cast<std::uint64_t>(s.pitch)
                                                      : static_cast<std::uint64_t>(s.length);
            f[b + 2] = static_cast<std::uint64_t>(s.fstride);
        };
        for (std::size_t i = 0; i < u.in_ids.size(); ++i) put(static_cast<int>(i), u.in_ids[i]);
        for (std::size_t o = 0; o < u.out_ids.size(); ++o) put(static_cast<int>(u.in_ids.size() + o), u.out_ids[o]);
        f[f.size() - 4] = 0;                                  // first output row
        f[f.size() - 3] = static_cast<std::uint64_t>(u.height); // end row
        f[f.size() - 2] = reinterpret_cast<std::uint64_t>(scr);
        f[f.size() - 1] = np.scratch_bytes_per_frame;
        void* args[] = {f.data()};
        for (std::size_t ki = 0; ki < np.kernels.size(); ++ki) {
            const jit::KernelSpec& ks = np.kernels[ki];
            unsigned grid[3] = {1, 1, static_cast<unsigned>(frames)};
            unsigned block[3] = {static_cast<unsigned>(ks.block_x), static_cast<unsigned>(ks.block_y), 1};
            switch (ks.grid) {
            case jit::KernelSpec::Grid::Pixels:
            case jit::KernelSpec::Grid::OutPixels:
                grid[0] = static_cast<unsigned>((u.width + ks.block_x * ks.cols - 1) / (ks.block_x * ks.cols));
                grid[1] = static_cast<unsigned>((u.height + ks.block_y * ks.rows - 1) / (ks.block_y * ks.rows));
                break;
            case jit::KernelSpec::Grid::Strided: {
                grid[0] = static_cast<unsigned>((u.width + ks.block_x - 1) / ks.block_x);
                const long long rows = (u.height + ks.block_y - 1) / ks.block_y;
                const long long want = std::max<long long>(1, 1184 / (static_cast<long long>(grid[0]) * frames));
                grid[1] = static_cast<unsigned>(std::max<long long>(1, std::min(rows, want)));
                break;
            }
            case jit::KernelSpec::Grid::Single: block[1] = 1; break;
            case jit::KernelSpec::Grid::Rows: grid[0] = static_cast<unsigned>((u.height + 127) / 128); break;
            case jit::KernelSpec::Grid::Cols: grid[0] = static_cast<unsigned>((u.width + 127) / 128); break;
            }
            dev::check(gvxb_jit_launch(ctx, u.module, static_cast<int>(ki), grid, block, 0, args), "generated kernel launch");
        }
    }

    void upload(ObjectId id, const Buffer& b, int frame) {
        const dev::ObjInfo& oi = prog->objects.at(id);
        Store& s = ensure(id);
        char* base = static_cast<char*>(s.ptr) + static_cast<std::int64_t>(frame) * s.fstride;
        if (oi.desc.kind == ObjKind::Image) {
            const std::size_t row = static_cast<std::size_t>(oi.desc.width) * bytes_per_pixel(oi.desc.format);
            if (b.bytes.size() < row * oi.desc.height) throw Error(ErrorCode::ShapeMismatch, "image payload too small", id);
            int pinned = 0;
            if (staging && row * oi.desc.height > Staging::kChunk / 4) gvxb_host_is_pinned(b.bytes.data(), &pinned);
            static const bool trace = std::getenv("GVX_TRACE_HOST") != nullptr;
            if (trace) std::fprintf(stderr, "[gvx host] upload object %llu (%p, %zu B): %s%s\n",
                                    static_cast<unsigned long long>(id), static_cast<const void*>(b.bytes.data()),
                                    row * static_cast<std::size_t>(oi.desc.height),
                                    pinned ? "page-locked, direct DMA" : "pageable, staged",
                                    fill && fill->id == id ? ", filled chunk-wise" : "");
            if (fill && fill->id == id && fill->src) {
                // the facade's input Buffer is filled from the caller's frame here
                auto* dst = const_cast<std::uint8_t*>(b.bytes.data());
                const std::size_t total = row * static_cast<std::size_t>(oi.desc.height);
                if (pinned && s.pitch == static_cast<std::int64_t>(row)) {
                    // chunk by chunk, each chunk's DMA overlapping the next copy
                    constexpr std::size_t kFill = std::size_t(2) << 20;
                    for (std::size_t o = 0; o < total; o += kFill) {
                        const std::size_t n = std::min(kFill, total - o);
                        dev::parallel_copy(dst + o, fill->src + o, n, /*streaming=*/true);
                        dev::check(gvxb_upload_2d(ctx, base + o, n, dst + o, n, n, 1), "image upload");
                    }
                    return;
                }
                dev::parallel_copy(dst, fill->src, total, /*streaming=*/true);
            }
            if (staging && !pinned && row * oi.desc.height > Staging::kChunk / 4) {
                staging->upload(base, static_cast<std::size_t>(s.pitch), b.bytes.data(), row,
                                static_cast<std::size_t>(oi.desc.height));
                return;
            }
            dev::check(gvxb_upload_2d(ctx, base, static_cast<std::size_t>(s.pitch), b.bytes.data(), row, row,
                                      static_cast<std::size_t>(oi.desc.height)),
                       "image upload");
            return;
        }
        std::vector<gvxb_value> vals;
        auto push = [&](const Value& v) {
            gvxb_value g;
            g.real = v.real ? 1 : 0;
            if (v.real) std::memcpy(&g.bits, &v.f, 8);
            else g.bits = v.i;
            vals.push_back(g);
        };
        if (oi.desc.kind == ObjKind::Scalar) {
            push(b.scalar);
        } else if (b.has_dist) {
            for (std::int64_t c : b.dist.counts) push(Value::of_int(c));
        } else {
            for (const Value& v : b.elements) push(v);
        }
        const int cap = static_cast<int>(s.fstride / 16);
        if (static_cast<int>(vals.size()) > cap) {
            if (!s.owned) throw Error(ErrorCode::ShapeMismatch, "array payload exceeds bound storage", id);
            gvxb_sync(ctx);
            gvxb_free(ctx, s.ptr);
            s.fstride = static_cast<std::int64_t>(vals.size()) * 16;
            dev::check(gvxb_alloc(ctx, static_cast<std::size_t>(s.fstride) * frames, &s.ptr), "device allocation");
            base = static_cast<char*>(s.ptr) + static_cast<std::int64_t>(frame) * s.fstride;
        }
        if (oi.desc.kind != ObjKind::Scalar) s.length = static_cast<int>(vals.size());
        if (!vals.empty())
            dev::check(gvxb_upload_2d(ctx, base, vals.size() * 16, vals.data(), vals.size() * 16, vals.size() * 16, 1),
                       "value upload");
    }

    Buffer download(ObjectId id, int frame) {
        const dev::ObjInfo& oi = prog->objects.at(id);
        Store& s = ensure(id);
        const char* base = static_cast<const char*>(s.ptr) + static_cast<std::int64_t>(frame) * s.fstride;
        Buffer b;
        b.id = id;
        b.desc = exec_graph->resolved().count(id) ? exec_graph->desc(id) : oi.desc;
        if (oi.desc.kind == ObjKind::Image) {
            const std::size_t row = static_cast<std::size_t>(oi.desc.width) * bytes_per_pixel(oi.desc.format);
            if (out_pool) { // a recycled page-locked vector: DMA straight into it
                auto it = out_pool->find(id);
                if (it != out_pool->end() && it->second.size() == row * static_cast<std::size_t>(oi.desc.height)) {
                    const ResolvedDesc d = b.desc;
                    b = Buffer{};
                    b.id = id;
                    b.desc = d;
                    b.bytes = std::move(it->second);
                    out_pool->erase(it);
                    dev::check(gvxb_download_2d(ctx, b.bytes.data(), row, base, static_cast<std::size_t>(s.pitch), row,
                                                static_cast<std::size_t>(oi.desc.height)),
                               "image download");
                    dev::check(gvxb_sync(ctx), "download sync");
                    return b;
                }
            }
            b = Buffer::image(b.desc);
            b.id = id;
            if (staging && row * oi.desc.height > Staging::kChunk / 4) {
                staging->download(b.bytes.data(), base, static_cast<std::size_t>(s.pitch), row,
                                  static_cast<std::size_t>(oi.desc.height));
                return b;
            }
            dev::check(gvxb_download_2d(ctx, b.bytes.data(), row, base, static_cast<std::size_t>(s.pitch), row,
                                        static_cast<std::size_t>(oi.desc.height)),
                       "image download");
            dev::check(gvxb_sync(ctx), "download sync");
            return b;
        }
        int n = oi.desc.kind == ObjKind::Scalar ? 1 : oi.length;
        if (oi.role == dev::ArrayRole::Distribution) n = oi.bins;
        if (oi.role == dev::ArrayRole::Location) n = 2;
        std::vector<gvxb_value> vals(static_cast<std::size_t>(std::max(n, 0)));
        if (!vals.empty())
            dev::check(gvxb_download_2d(ctx, vals.data(), vals.size() * 16, base, vals.size() * 16, vals.size() * 16, 1),
                       "value download");
        dev::check(gvxb_sync(ctx), "download sync");
        auto value = [](const gvxb_value& g) {
            if (!g.real) return Value::of_int(g.bits);
            double d;
            std::memcpy(&d, &g.bits, 8);
            return Value::of_real(d);
        };
        if (oi.desc.kind == ObjKind::Scalar) {
            b.scalar = value(vals[0]);
        } else if (oi.role == dev::ArrayRole::Distribution) {
            b.has_dist = true;
            b.dist.bins = oi.bins;
            b.dist.offset = oi.offset;
            b.dist.range = oi.range;
            for (const gvxb_value& g : vals) b.dist.counts.push_back(g.bits);
        } else {
            for (const gvxb_value& g : vals) b.elements.push_back(value(g));
        }
        return b;
    }

    void run_all() {
        for (std::size_t i = 0; i < prog->units.size(); ++i) launch_unit(i);
    }
};

namespace {

std::map<ObjectId, std::vector<Value>> matrix_inputs(const VerifiedGraph& vg, const InputMap* inputs) {
    std::map<ObjectId, std::vector<Value>> m;
    const Context& ctx = vg.context();
    for (ObjectId id : vg.graph().data()) {
        const DataObject* o = ctx.find(id);
        if (!o || o->kind != ObjKind::Matrix) continue;
        if (inputs) {
            auto it = inputs->find(id);
            if (it != inputs->end()) {
                m[id] = it->second.elements;
                continue;
            }
        }
        m[id] = o->matrix_values;
    }
    return m;
}

std::string program_key(std::uint64_t stamp, bool naive, const std::map<ObjectId, std::vector<Value>>& mats) {
    std::ostringstream os;
    os << (naive ? "n" : "p") << stamp;
    for (const auto& [id, vals] : mats) {
        os << "|" << id << ":";
        for (const Value& v : vals) os << (v.real ? "r" : "i") << (v.real ? v.f : static_cast<double>(v.i)) << ",";
    }
    return os.str();
}

std::mutex g_prog_mu;
std::map<std::string, std::shared_ptr<dev::Program>>& program_cache() {
    static auto* c = new std::map<std::string, std::shared_ptr<dev::Program>>();
    return *c;
}

std::shared_ptr<dev::Program> cached_program(const std::string& key, const std::function<std::shared_ptr<dev::Program>()>& make) {
    {
        std::lock_guard<std::mutex> lock(g_prog_mu);
        auto it = program_cache().find(key);
        if (it != program_cache().end()) return it->second;
    }
    auto p = make();
    std::lock_guard<std::mutex> lock(g_prog_mu);
    if (program_cache().size() > 256) program_cache().clear();
    return program_cache().emplace(key, p).first->second;
}

std::shared_ptr<dev::Program> naive_program(const VerifiedGraph& g, const InputMap* inputs) {
    auto mats = matrix_inputs(g, inputs);
    return cached_program(program_key(g.stamp(), true, mats), [&] { return dev::build_naive(g, mats); });
}

std::shared_ptr<dev::Program> plan_program(const OptimizedPlan& plan, const InputMap* inputs) {
    auto mats = matrix_inputs(plan.fused, inputs);
    auto base_mats = matrix_inputs(plan.base, inputs);
    mats.insert(base_mats.begin(), base_mats.end());
    return cached_program(program_key(plan.fused.stamp(), false, mats), [&] { return dev::build_plan(plan, mats); });
}

} // namespace

std::shared_ptr<dev::Program> dev::program_of(const OptimizedPlan& plan) { return plan_program(plan, nullptr); }

namespace {

/// The reference's input binding rules (ref:src/execute.cpp:300-346).
std::map<ObjectId, const Buffer*> bind_inputs(const VerifiedGraph& vg, const InputMap& inputs,
                                               std::map<ObjectId, Buffer>& defaults) {
    const AppGraph& g = vg.graph();
    const Context& ctx = vg.context();
    for (const auto& [id, buf] : inputs) {
        const DataObject* o = ctx.find(id);
        if (!o) throw Error(ErrorCode::UnknownObject, "input #" + std::to_string(id), id);
        if (o->is_virtual)
            throw Error(ErrorCode::AccessDenied, "virtual object '" + o->name + "' cannot be written from the host", id);
    }
    std::map<ObjectId, const Buffer*> bound;
    for (ObjectId id : g.data()) {
        const DataObject* o = ctx.find(id);
        if (!o || o->is_virtual || g.producer(id) != kInvalidId) continue;
        auto it = inputs.find(id);
        if (it != inputs.end()) {
            const ResolvedDesc& want = vg.desc(id);
            const Buffer& got = it->second;
            if (want.kind != got.desc.kind ||
                (want.kind == ObjKind::Image &&
                 (want.width != got.desc.width || want.height != got.desc.height || want.format != got.desc.format)))
                throw Error(ErrorCode::ShapeMismatch, "input '" + o->name + "' does not match its declaration", id);
            bound[id] = &got;
            continue;
        }
        if (o->kind == ObjKind::Scalar && o->scalar_value) {
            Buffer b = Buffer::scalar_value(o->element_type, *o->scalar_value);
            b.id = id;
            b.desc = vg.desc(id);
            bound[id] = &(defaults[id] = b);
            continue;
        }
        if (o->kind == ObjKind::Matrix && !o->matrix_values.empty()) {
            Buffer b;
            b.id = id;
            b.desc = vg.desc(id);
            b.elements = o->matrix_values;
            bound[id] = &(defaults[id] = b);
            continue;
        }
        if (!g.consumers(id).empty())
            throw Error(ErrorCode::MissingInput, "no buffer for input '" + o->name + "'", id);
    }
    return bound;
}

struct HostSession {
    std::mutex mu;
    DeviceSession::Impl impl;
    /// large frames of single-group stencil / point programs: row pieces
    /// pipelined from host memory (built on first use; null = not eligible)
    std::unique_ptr<BandedSession> pieces;
    bool pieces_tried = false;
};

/// Output rows per piece for the pipelined host path, or 0 to run the frame
/// whole (small frames: the per-piece transfer and launch overheads win).
int host_piece_rows(const dev::Program& prog, ObjectId input, int height) {
    static const char* off = std::getenv("GVX_HOST_PIECES");
    if (off && off[0] == '0') return 0;
    const dev::ObjInfo& oi = prog.objects.at(input);
    const std::size_t bytes =
        static_cast<std::size_t>(oi.desc.width) * bytes_per_pixel(oi.desc.format) * static_cast<std::size_t>(height);
    static const std::size_t min_bytes = [] {
        const char* e = std::getenv("GVX_HOST_PIECE_MIN_BYTES");
        return e ? static_cast<std::size_t>(std::atoll(e)) : (std::size_t(1) << 20);
    }();
    if (bytes < min_bytes || height < 256) return 0;
    if (const char* e = std::getenv("GVX_HOST_PIECE_ROWS")) return std::max(16, std::atoi(e));
    // four pieces: measured best of 2 / 3 / 4 / 6 / 8 / 16 on cfg1, 2, 3 and 5
    // (the host copies of the pieces are the critical path; each extra piece
    // adds a wait on its download before its rows can be copied out)
    return (height + 3) / 4;
}

/// Device storage is kept per program between synchronous host runs (the
/// reference allocates per run; reusing it keeps run_plan at copy speed).
std::shared_ptr<HostSession> host_session(const std::shared_ptr<dev::Program>& prog) {
    static std::mutex mu;
    static auto& cache =
        *new std::map<const dev::Program*, std::pair<std::weak_ptr<dev::Program>, std::shared_ptr<HostSession>>>();
    std::lock_guard<std::mutex> lock(mu);
    for (auto it = cache.begin(); it != cache.end();)
        it = it->second.first.expired() ? cache.erase(it) : std::next(it);
    auto& slot = cache[prog.get()];
    if (!slot.second) {
        slot.first = prog;
        slot.second = std::make_shared<HostSession>();
        slot.second->impl.prog = prog;
        slot.second->impl.frames = 1;
        slot.second->impl.ctx = dev::own_context();
        slot.second->impl.owns_ctx = true;
        slot.second->impl.staging = std::make_unique<Staging>(slot.second->impl.ctx);
    }
    return slot.second;
}

ExecutionReport execute(const std::shared_ptr<dev::Program>& prog, const VerifiedGraph& vg, const InputMap& inputs,
                        std::map<ObjectId, std::vector<std::uint8_t>>* out_pool = nullptr,
                        const detail::HostFill* fill = nullptr) {
    std::map<ObjectId, Buffer> defaults;
    auto bound = bind_inputs(vg, inputs, defaults);

    std::shared_ptr<HostSession> hs = host_session(prog);
    std::lock_guard<std::mutex> lock(hs->mu);
    DeviceSession::Impl& s = hs->impl;
    s.exec_graph = &vg;
    s.out_pool = out_pool;
    s.fill = fill;
    struct PoolReset {
        DeviceSession::Impl& s;
        ~PoolReset() {
            s.out_pool = nullptr;
            s.fill = nullptr;
        }
    } pool_reset{s};
    static const bool trace = std::getenv("GVX_TRACE_HOST") != nullptr;
    using clock = std::chrono::steady_clock;
    const auto t0 = clock::now();
    if (!hs->pieces_tried) {
        hs->pieces_tried = true;
        hs->pieces = detail::whole_image_band(prog);
    }
    if (hs->pieces) {
        const ObjectId in_id = detail::whole_image_band_input(*hs->pieces);
        const int H = prog->objects.at(in_id).desc.height;
        const int piece = host_piece_rows(*prog, in_id, H);
        auto bit = bound.find(in_id);
        if (piece > 0 && bit != bound.end()) {
            // row pieces: each piece's input rows go up, its kernel runs and its
            // output rows come down while the host copies of its neighbours run
            const Buffer& ib = *bit->second;
            const dev::ObjInfo& ii = prog->objects.at(in_id);
            const std::size_t in_bytes =
                static_cast<std::size_t>(ii.desc.width) * bytes_per_pixel(ii.desc.format) * ii.desc.height;
            if (ib.bytes.size() < in_bytes) throw Error(ErrorCode::ShapeMismatch, "image payload too small", in_id);
            BandedSession::HostRows in_rows;
            in_rows.id = in_id;
            if (fill && fill->id == in_id && fill->src) {
                in_rows.host = const_cast<std::uint8_t*>(fill->src);
            } else {
                in_rows.host = const_cast<std::uint8_t*>(ib.bytes.data());
                int pinned = 0;
                gvxb_host_is_pinned(ib.bytes.data(), &pinned);
                in_rows.page_locked = pinned != 0;
            }
            ExecutionReport report;
            std::vector<BandedSession::HostRows> outs;
            const AppGraph& g = vg.graph();
            const Context& gctx = vg.context();
            for (ObjectId id : g.data()) {
                const DataObject* o = gctx.find(id);
                if (!o || o->is_virtual || g.producer(id) == kInvalidId || !prog->objects.count(id)) continue;
                const dev::ObjInfo& oi = prog->objects.at(id);
                const std::size_t bytes =
                    static_cast<std::size_t>(oi.desc.width) * bytes_per_pixel(oi.desc.format) * oi.desc.height;
                Buffer b;
                const ResolvedDesc d = vg.resolved().count(id) ? vg.desc(id) : oi.desc;
                BandedSession::HostRows r;
                r.id = id;
                auto pit = out_pool ? out_pool->find(id) : decltype(out_pool->end()){};
                if (out_pool && pit != out_pool->end() && pit->second.size() == bytes) {
                    b.desc = d;
                    b.bytes = std::move(pit->second);
                    out_pool->erase(pit);
                    r.page_locked = true;
                    if (fill && fill->drain_id == id && fill->drain_dst) {
                        r.drain = fill->drain_dst;
                        fill->drained = true;
                    }
                } else {
                    b = Buffer::image(d);
                }
                b.id = id;
                Buffer& slot = report.outputs[id] = std::move(b);
                r.host = slot.bytes.data();
                outs.push_back(r);
            }
            const long long launches0 = detail::whole_image_band_launches(*hs->pieces);
            const long long dyn = hs->pieces->run_host_rows(in_rows, outs, piece);
            report.counters.kernel_launches = detail::whole_image_band_launches(*hs->pieces) - launches0;
            report.counters.pixels_read = dyn;
            for (const dev::Unit& u : prog->units) {
                report.counters.pixels_read += u.static_reads;
                report.counters.pixels_written += u.static_writes;
            }
            if (trace)
                std::fprintf(stderr, "[gvx host] %d-row pieces: %.1f us\n", piece,
                             std::chrono::duration<double, std::micro>(clock::now() - t0).count());
            return report;
        }
    }
    gvxb_ctx_set_stream(s.ctx, nullptr);
    if (s.scratch.size() != prog->units.size()) s.prepare();
    for (const auto& [id, b] : bound)
        if (prog->objects.count(id)) s.upload(id, *b, 0);
    if (trace) gvxb_sync(s.ctx); // attribute the H2D DMA to the upload phase
    const auto t1 = clock::now();
    dev::check(gvxb_status_reset(s.ctx), "status reset");
    const std::int64_t launches0 = gvxb_launch_count(s.ctx);
    s.run_all();
    const auto t1b = clock::now();
    std::uint32_t status = 0;
    long long dyn_reads = 0;
    dev::check(gvxb_status_counter_read(s.ctx, &status, &dyn_reads), "device status");
    if (status & GVXB_STATUS_DIV_BY_ZERO) throw Error(ErrorCode::DivByZero, "division by zero");
    if (status & GVXB_STATUS_INDEX_RANGE) throw Error(ErrorCode::ShapeMismatch, "array index out of range");
    const auto t2 = clock::now();

    ExecutionReport report;
    report.counters.kernel_launches = gvxb_launch_count(s.ctx) - launches0;
    report.counters.pixels_read = dyn_reads;
    for (const dev::Unit& u : prog->units) {
        report.counters.pixels_read += u.static_reads;
        report.counters.pixels_written += u.static_writes;
    }
    const AppGraph& g = vg.graph();
    const Context& ctx = vg.context();
    for (ObjectId id : g.data()) {
        const DataObject* o = ctx.find(id);
        if (!o || o->is_virtual || g.producer(id) == kInvalidId) continue;
        if (!prog->objects.count(id)) continue;
        report.outputs[id] = s.download(id, 0);
    }
    if (trace) {
        const auto t3 = clock::now();
        auto us = [](clock::duration d) { return std::chrono::duration<double, std::micro>(d).count(); };
        std::fprintf(stderr, "[gvx host] upload %.1f us, launch (host) %.1f us, device+status %.1f us, download %.1f us\n",
                     us(t1 - t0), us(t1b - t1), us(t2 - t1b), us(t3 - t2));
    }
    return report;
}

} // namespace

namespace detail {

ExecutionReport run_naive_pooled(const VerifiedGraph& g, const InputMap& inputs,
                                 std::map<ObjectId, std::vector<std::uint8_t>>* out_pool, const HostFill* fill) {
    if (!g.stamped()) throw Error(ErrorCode::UnstampedGraph, "execution needs a verified graph");
    auto prog = naive_program(g, &inputs);
    ExecutionReport r = execute(prog, g, inputs, out_pool, fill);
    r.counters.transfers_executed = static_cast<std::int64_t>(g.graph().nodes().size()) * 2;
    return r;
}

ExecutionReport run_plan_pooled(const OptimizedPlan& plan, const InputMap& inputs,
                                std::map<ObjectId, std::vector<std::uint8_t>>* out_pool, const HostFill* fill) {
    if (!plan.fused.stamped()) throw Error(ErrorCode::UnstampedGraph, "plan execution needs a verified fused graph");
    auto prog = plan_program(plan, &inputs);
    ExecutionReport r = execute(prog, plan.fused, inputs, out_pool, fill);
    r.counters.transfers_executed = plan.transfers.optimized_count();
    return r;
}

} // namespace detail

ExecutionReport run_naive(const VerifiedGraph& g, const InputMap& inputs) {
    return detail::run_naive_pooled(g, inputs, nullptr, nullptr);
}

ExecutionReport run_plan(const OptimizedPlan& plan, const InputMap& inputs) {
    return detail::run_plan_pooled(plan, inputs, nullptr, nullptr);
}

// ------------------------------------------------------------ DeviceSession

DeviceSession::DeviceSession(const OptimizedPlan& plan, int frames) : impl_(std::make_unique<Impl>()) {
    if (!plan.fused.stamped()) throw Error(ErrorCode::UnstampedGraph, "plan execution needs a verified fused graph");
    impl_->prog = plan_program(plan, nullptr);
    impl_->exec_copy = plan.fused;
    impl_->exec_graph = &impl_->exec_copy;
    impl_->frames = std::max(1, frames);
    impl_->ctx = dev::own_context();
    impl_->owns_ctx = true;
}

DeviceSession::DeviceSession(const VerifiedGraph& g, int frames) : impl_(std::make_unique<Impl>()) {
    if (!g.stamped()) throw Error(ErrorCode::UnstampedGraph, "execution needs a verified graph");
    impl_->prog = naive_program(g, nullptr);
    impl_->exec_copy = g;
    impl_->exec_graph = &impl_->exec_copy;
    impl_->frames = std::max(1, frames);
    impl_->ctx = dev::own_context();
    impl_->owns_ctx = true;
}

DeviceSession::~DeviceSession() = default;

void DeviceSession::bind(ObjectId id, DeviceTensor t) {
    auto it = impl_->prog->objects.find(id);
    if (it == impl_->prog->objects.end()) return; // not touched by the program
    if (it->second.is_virtual) throw Error(ErrorCode::AccessDenied, "virtual objects are program-internal", id);
    Impl::Store s;
    s.ptr = t.data;
    s.pitch = t.pitch;
    const ResolvedDesc& d = it->second.desc;
    if (d.kind == ObjKind::Image) {
        if (t.pitch % 16 != 0) throw Error(ErrorCode::ShapeMismatch, "device image pitch must be a multiple of 16", id);
        s.fstride = t.frame_stride ? t.frame_stride : t.pitch * d.height;
    } else {
        s.length = d.kind == ObjKind::Scalar ? 1 : std::max(it->second.length, 1);
        s.fstride = t.frame_stride ? t.frame_stride : static_cast<std::int64_t>(s.length) * 16;
    }
    auto old = impl_->store.find(id);
    if (old != impl_->store.end() && old->second.owned) gvxb_free(impl_->ctx, old->second.ptr);
    impl_->store[id] = s;
}

DeviceTensor DeviceSession::tensor(ObjectId id) {
    Impl::Store& s = impl_->ensure(id);
    return DeviceTensor{s.ptr, s.pitch, s.fstride};
}

void DeviceSession::set_stream(void* s) {
    impl_->stream = s;
    gvxb_ctx_set_stream(impl_->ctx, s); // the session's own context: kept until changed
}

void DeviceSession::set_overlap(int mode) { dev::check(gvxb_ctx_set_overlap(impl_->ctx, mode), "set overlap"); }

void DeviceSession::launch() {
    if (impl_->scratch.size() != impl_->prog->units.size()) impl_->prepare();
    const std::int64_t n0 = gvxb_launch_count(impl_->ctx);
    impl_->run_all();
    impl_->last_launches = static_cast<int>(gvxb_launch_count(impl_->ctx) - n0);
}

void DeviceSession::synchronize() {
    std::uint32_t status = 0;
    const int rc = gvxb_status_read(impl_->ctx, &status);
    dev::check(rc, "device status");
    if (status & GVXB_STATUS_DIV_BY_ZERO) throw Error(ErrorCode::DivByZero, "division by zero");
    if (status & GVXB_STATUS_INDEX_RANGE) throw Error(ErrorCode::ShapeMismatch, "array index out of range");
}

void DeviceSession::upload(ObjectId id, const Buffer& b, int frame) {
    if (!impl_->prog->objects.count(id)) return;
    impl_->upload(id, b, frame);
}

Buffer DeviceSession::download(ObjectId id, int frame) {
    if (!impl_->prog->objects.count(id)) throw Error(ErrorCode::UnknownObject, "object not produced on the device", id);
    Buffer b = impl_->download(id, frame);
    return b;
}

int DeviceSession::frames() const { return impl_->frames; }
int DeviceSession::launches_per_run() const {
    // what the last execution launched (conv+stats picks its one- or
    // three-launch form in the C-ABI), else the program's estimate
    return impl_->last_launches > 0 ? impl_->last_launches : impl_->prog->launches_per_run(impl_->frames);
}
std::string DeviceSession::describe() const { return impl_->prog->describe(); }

// ------------------------------------------------------------ HostPipeline

struct HostPipeline::Impl {
    struct Slot {
        DeviceSession::Impl s; // device storage + lowered program; s.ctx = own context
        void* done = nullptr;  // event after the slot's last download
        void* pin_status = nullptr;
        std::map<ObjectId, void*> pin;         // page-locked staging per image object
        std::map<ObjectId, std::size_t> bytes; // its size
        std::vector<ObjectId> image_outs, other_outs;
        std::int64_t launches0 = 0;
        bool busy = false;
        ~Slot() { // device storage and the context go with `s`
            if (!s.ctx) return;
            gvxb_sync(s.ctx);
            if (done) gvxb_event_destroy(done);
            if (pin_status) gvxb_host_free(pin_status);
            for (auto& kv : pin) gvxb_host_free(kv.second);
        }
    };
    std::shared_ptr<dev::Program> prog;
    VerifiedGraph exec;
    std::int64_t transfers = 0;
    std::vector<std::unique_ptr<Slot>> slots;
    std::deque<int> inflight; // slot indices in submission order
    std::deque<ExecutionReport> ready;
    int next_slot = 0;
    const void* last_view = nullptr;
    std::vector<std::uint8_t> view_hold;

    void init(int depth) {
        dev::context(); // device check + the shared NVRTC modules
        int device = 0;
        if (const char* e = std::getenv("GVX_DEVICE")) device = std::atoi(e);
        for (int i = 0; i < std::max(1, depth); ++i) {
            auto sl = std::make_unique<Slot>();
            sl->s.prog = prog;
            sl->s.exec_graph = &exec;
            sl->s.frames = 1;
            dev::check(gvxb_ctx_create(device, &sl->s.ctx), "pipeline context");
            sl->s.owns_ctx = true;
            dev::check(gvxb_event_create(&sl->done), "pipeline event");
            dev::check(gvxb_host_alloc(32, &sl->pin_status), "pipeline status staging");
            sl->s.prepare();
            const AppGraph& g = exec.graph();
            const Context& ctx = exec.context();
            for (ObjectId id : g.data()) {
                const DataObject* o = ctx.find(id);
                if (!o || o->is_virtual || g.producer(id) == kInvalidId || !prog->objects.count(id)) continue;
                (prog->objects.at(id).desc.kind == ObjKind::Image ? sl->image_outs : sl->other_outs).push_back(id);
            }
            slots.push_back(std::move(sl));
        }
    }

    void* staging(Slot& sl, ObjectId id, std::size_t n) {
        auto it = sl.pin.find(id);
        if (it != sl.pin.end() && sl.bytes[id] >= n) return it->second;
        if (it != sl.pin.end()) gvxb_host_free(it->second);
        void* p = nullptr;
        dev::check(gvxb_host_alloc(n, &p), "pipeline staging");
        sl.pin[id] = p;
        sl.bytes[id] = n;
        return p;
    }

    void complete_oldest(ObjectId direct = kInvalidId, void* dst = nullptr, std::size_t dst_bytes = 0) {
        const int k = inflight.front();
        inflight.pop_front();
        Slot& sl = *slots[static_cast<std::size_t>(k)];
        dev::check(gvxb_event_sync(sl.done), "pipeline wait");
        sl.busy = false;
        std::uint64_t st[2];
        std::memcpy(st, sl.pin_status, sizeof st);
        if (st[0] & GVXB_STATUS_DIV_BY_ZERO) throw Error(ErrorCode::DivByZero, "division by zero");
        if (st[0] & GVXB_STATUS_INDEX_RANGE) throw Error(ErrorCode::ShapeMismatch, "array index out of range");
        ExecutionReport r;
        r.counters.kernel_launches = gvxb_launch_count(sl.s.ctx) - sl.launches0;
        r.counters.pixels_read = static_cast<std::int64_t>(st[1]);
        for (const dev::Unit& u : prog->units) {
            r.counters.pixels_read += u.static_reads;
            r.counters.pixels_written += u.static_writes;
        }
        r.counters.transfers_executed = transfers;
        for (ObjectId id : sl.image_outs) {
            const dev::ObjInfo& oi = prog->objects.at(id);
            if (id == direct) {
                if (!dst) { // view: the caller reads the staging in place
                    last_view = sl.pin.at(id);
                    continue;
                }
                const std::size_t n = static_cast<std::size_t>(oi.desc.width) * bytes_per_pixel(oi.desc.format) *
                                      static_cast<std::size_t>(oi.desc.height);
                if (dst_bytes < n) throw Error(ErrorCode::ShapeMismatch, "output buffer too small", id);
                dev::parallel_copy(dst, sl.pin.at(id), n);
                continue;
            }
            Buffer b = Buffer::image(exec.resolved().count(id) ? exec.desc(id) : oi.desc);
            b.id = id;
            dev::parallel_copy(b.bytes.data(), sl.pin.at(id), b.bytes.size());
            r.outputs[id] = std::move(b);
        }
        for (ObjectId id : sl.other_outs) r.outputs[id] = sl.s.download(id, 0); // small: values / counts
        ready.push_back(std::move(r));
    }

    /// Stages the frame through the slot's page-locked buffer, or (direct)
    /// DMAs it from the caller's page-locked memory.
    void upload_image(Slot& sl, ObjectId id, const void* data, std::size_t bytes, bool direct = false) {
        const dev::ObjInfo& oi = prog->objects.at(id);
        const std::size_t row = static_cast<std::size_t>(oi.desc.width) * bytes_per_pixel(oi.desc.format);
        const std::size_t n = row * static_cast<std::size_t>(oi.desc.height);
        if (bytes < n) throw Error(ErrorCode::ShapeMismatch, "image payload too small", id);
        const void* from = data;
        if (direct) {
            int pinned = 0;
            dev::check(gvxb_host_is_pinned(data, &pinned), "pinned query");
            if (!pinned) throw Error(ErrorCode::BadFormat, "submit_pinned: input is not page-locked host memory", id);
        } else {
            void* pin = staging(sl, id, n);
            dev::parallel_copy(pin, data, n, /*streaming=*/true);
            from = pin;
        }
        DeviceSession::Impl::Store& st = sl.s.ensure(id);
        dev::check(gvxb_upload_2d(sl.s.ctx, st.ptr, static_cast<std::size_t>(st.pitch), from, row, row,
                                  static_cast<std::size_t>(oi.desc.height)),
                   "pipeline upload");
    }

    /// The slot the next frame uses (round robin = submission order): when
    /// every slot is in flight, the oldest completes first.
    Slot& take_slot() {
        if (static_cast<int>(inflight.size()) >= static_cast<int>(slots.size())) complete_oldest();
        return *slots[static_cast<std::size_t>(next_slot)];
    }

    static double us_since(std::chrono::steady_clock::time_point t) {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t).count();
    }

    void submit_raw(ObjectId id, const void* data, std::size_t bytes, bool direct = false) {
        static const bool trace = std::getenv("GVX_TRACE_HOST") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        InputMap none;
        std::map<ObjectId, Buffer> defaults;
        // the graph's other inputs (bound scalars / matrices) as run_plan binds them
        InputMap probe;
        Buffer placeholder;
        placeholder.id = id;
        placeholder.desc = exec.desc(id);
        probe[id] = placeholder;
        auto bound = bind_inputs(exec, probe, defaults);
        Slot& sl = take_slot();
        const double t_take = trace ? us_since(t0) : 0;
        for (const auto& [oid, b] : bound) {
            if (oid == id || !prog->objects.count(oid)) continue;
            if (prog->objects.at(oid).desc.kind == ObjKind::Image)
                throw Error(ErrorCode::MissingInput, "the raw-pointer submit takes a graph with one image input", oid);
            sl.s.upload(oid, *b, 0);
        }
        if (prog->objects.count(id)) upload_image(sl, id, data, bytes, direct);
        const double t_up = trace ? us_since(t0) : 0;
        launch_slot(sl);
        if (trace)
            std::fprintf(stderr, "[gvx pipeline] submit: take %.1f us, copy+upload %.1f us, launch %.1f us\n", t_take,
                         t_up - t_take, us_since(t0) - t_up);
    }

    void submit(const InputMap& inputs) {
        std::map<ObjectId, Buffer> defaults;
        auto bound = bind_inputs(exec, inputs, defaults);
        Slot& sl = take_slot();
        for (const auto& [id, b] : bound) {
            if (!prog->objects.count(id)) continue;
            if (prog->objects.at(id).desc.kind != ObjKind::Image) sl.s.upload(id, *b, 0);
            else upload_image(sl, id, b->bytes.data(), b->bytes.size());
        }
        launch_slot(sl);
    }

    void launch_slot(Slot& sl) {
        gvxb_ctx sctx = sl.s.ctx;
        dev::check(gvxb_status_reset(sctx), "status reset");
        sl.launches0 = gvxb_launch_count(sctx);
        sl.s.run_all();
        for (ObjectId id : sl.image_outs) {
            const dev::ObjInfo& oi = prog->objects.at(id);
            const std::size_t row = static_cast<std::size_t>(oi.desc.width) * bytes_per_pixel(oi.desc.format);
            void* pin = staging(sl, id, row * static_cast<std::size_t>(oi.desc.height));
            DeviceSession::Impl::Store& st = sl.s.ensure(id);
            dev::check(gvxb_download_2d(sctx, pin, row, st.ptr, static_cast<std::size_t>(st.pitch), row,
                                        static_cast<std::size_t>(oi.desc.height)),
                       "pipeline download");
        }
        std::uint32_t* status = nullptr;
        dev::check(gvxb_status_ptr(sctx, &status), "status pointer");
        dev::check(gvxb_download_2d(sctx, sl.pin_status, 16, status, 16, 16, 1), "status download");
        dev::check(gvxb_event_record(sctx, sl.done), "pipeline event");
        sl.busy = true;
        inflight.push_back(next_slot); // only once everything is enqueued
        next_slot = (next_slot + 1) % static_cast<int>(slots.size());
    }
};

HostPipeline::HostPipeline(const OptimizedPlan& plan, int depth) : impl_(std::make_unique<Impl>()) {
    if (!plan.fused.stamped()) throw Error(ErrorCode::UnstampedGraph, "plan execution needs a verified fused graph");
    impl_->prog = plan_program(plan, nullptr);
    impl_->exec = plan.fused;
    impl_->transfers = plan.transfers.optimized_count();
    impl_->init(depth);
}

HostPipeline::HostPipeline(const VerifiedGraph& g, int depth) : impl_(std::make_unique<Impl>()) {
    if (!g.stamped()) throw Error(ErrorCode::UnstampedGraph, "execution needs a verified graph");
    impl_->prog = naive_program(g, nullptr);
    impl_->exec = g;
    impl_->transfers = static_cast<std::int64_t>(g.graph().nodes().size()) * 2;
    impl_->init(depth);
}

HostPipeline::~HostPipeline() = default;

void HostPipeline::submit(const InputMap& inputs) { impl_->submit(inputs); }

void HostPipeline::submit(ObjectId image_input, const void* data, std::size_t bytes) {
    impl_->submit_raw(image_input, data, bytes);
}

void HostPipeline::submit_pinned(ObjectId image_input, const void* data, std::size_t bytes) {
    impl_->submit_raw(image_input, data, bytes, /*direct=*/true);
}

ExecutionReport HostPipeline::next_into(ObjectId image_output, void* dst, std::size_t bytes) {
    if (!impl_->ready.empty()) { // already completed into a Buffer (submit ran ahead)
        ExecutionReport r = std::move(impl_->ready.front());
        impl_->ready.pop_front();
        auto it = r.outputs.find(image_output);
        if (it != r.outputs.end()) {
            if (bytes < it->second.bytes.size()) throw Error(ErrorCode::ShapeMismatch, "output buffer too small");
            dev::parallel_copy(dst, it->second.bytes.data(), it->second.bytes.size());
            r.outputs.erase(it);
        }
        return r;
    }
    if (impl_->inflight.empty()) throw Error(ErrorCode::MissingInput, "no frame submitted");
    impl_->complete_oldest(image_output, dst, bytes);
    ExecutionReport r = std::move(impl_->ready.front());
    impl_->ready.pop_front();
    return r;
}

ExecutionReport HostPipeline::next() {
    if (impl_->ready.empty()) {
        if (impl_->inflight.empty()) throw Error(ErrorCode::MissingInput, "no frame submitted");
        impl_->complete_oldest();
    }
    ExecutionReport r = std::move(impl_->ready.front());
    impl_->ready.pop_front();
    return r;
}

ExecutionReport HostPipeline::next_view(ObjectId image_output, const void** view) {
    if (!impl_->ready.empty()) { // completed early into a Buffer: serve that copy
        ExecutionReport r = std::move(impl_->ready.front());
        impl_->ready.pop_front();
        auto it = r.outputs.find(image_output);
        if (it == r.outputs.end()) throw Error(ErrorCode::UnknownObject, "no such image output", image_output);
        impl_->view_hold = std::move(it->second.bytes);
        r.outputs.erase(it);
        *view = impl_->view_hold.data();
        return r;
    }
    if (impl_->inflight.empty()) throw Error(ErrorCode::MissingInput, "no frame submitted");
    impl_->last_view = nullptr;
    impl_->complete_oldest(image_output, nullptr, 0);
    ExecutionReport r = std::move(impl_->ready.front());
    impl_->ready.pop_front();
    if (!impl_->last_view) throw Error(ErrorCode::UnknownObject, "no such image output", image_output);
    *view = impl_->last_view;
    return r;
}

int HostPipeline::pending() const { return static_cast<int>(impl_->inflight.size() + impl_->ready.size()); }

int device_count() {
    int n = 0;
    return gvxb_device_count(&n) == GVXB_OK ? n : 0;
}

} // namespace gvx
