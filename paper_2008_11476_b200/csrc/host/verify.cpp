// vxVerifyGraph: structure + parameter checks and forward format propagation.
// Diagnostics, ordering and de-duplication follow ref:src/verify.cpp:82-351;
// the stamp comes from one process-wide counter (ref:src/verify.cpp:47-58)
// and doubles as the device-program cache key.
#include "graphvx/verify.hpp"

#include <algorithm>
#include <atomic>
#include <ostream>
#include <sstream>

namespace gvx {

const char* to_string(DiagCode c) {
    static const char* const names[] = {"CycleDetected",    "NotBipartite",    "UnboundParam",
                                        "DirectionMismatch", "FormatMismatch", "MultipleWriters",
                                        "UnresolvedVirtualFormat", "UnknownKernel"};
    auto i = static_cast<std::size_t>(c);
    return i < 8 ? names[i] : "?";
}

std::string Diagnostic::render() const {
    std::ostringstream os;
    os << to_string(code) << " object#";
    for (std::size_t i = 0; i < subjects.size(); ++i) os << (i ? "," : "") << subjects[i];
    os << ": " << message;
    return os.str();
}

std::ostream& operator<<(std::ostream& os, const Diagnostic& d) { return os << d.render(); }

const ResolvedDesc& VerifiedGraph::desc(ObjectId id) const {
    auto it = resolved_.find(id);
    if (it == resolved_.end())
        throw Error(ErrorCode::UnknownObject, "object #" + std::to_string(id) + " not resolved", id);
    return it->second;
}

struct VerifyAccess {
    static void seal(VerifiedGraph& vg, std::shared_ptr<const AppGraph> g, Context* ctx,
                     std::map<ObjectId, ResolvedDesc> resolved,
                     std::map<ObjectId, std::vector<ScalarType>> types, bool ok) {
        static std::atomic<std::uint64_t> next_stamp{1};
        vg.graph_ = std::move(g);
        vg.ctx_ = ctx;
        vg.resolved_ = std::move(resolved);
        vg.node_types_ = std::move(types);
        vg.stamp_ = ok ? next_stamp.fetch_add(1) : 0;
    }
};

namespace {

std::string describe(const ResolvedDesc& d) {
    if (d.kind == ObjKind::Image)
        return std::string(to_string(d.format)) + " " + std::to_string(d.width) + "x" +
               std::to_string(d.height);
    return to_string(d.element_type);
}

bool image_ready(const ResolvedDesc& d) {
    return d.format != ImageFormat::UNRESOLVED && d.width > 0;
}

class Checker {
public:
    explicit Checker(const AppGraph& g) : g_(g), ctx_(g.context()), reg_(ctx_.registry()) {}

    VerifyResult run() {
        structure();
        for (const OperatorNode& n : g_.nodes()) params(n);
        propagate();
        std::stable_sort(diags_.begin(), diags_.end(), [](const Diagnostic& a, const Diagnostic& b) {
            if (a.code != b.code) return a.code < b.code;
            const ObjectId x = a.subjects.empty() ? 0 : a.subjects.front();
            const ObjectId y = b.subjects.empty() ? 0 : b.subjects.front();
            return x < y;
        });
        diags_.erase(std::unique(diags_.begin(), diags_.end(),
                                 [](const Diagnostic& a, const Diagnostic& b) {
                                     return a.code == b.code && a.subjects == b.subjects &&
                                            a.message == b.message;
                                 }),
                     diags_.end());
        VerifyResult out;
        out.diagnostics = std::move(diags_);
        VerifyAccess::seal(out.verified, std::make_shared<AppGraph>(g_), &ctx_, std::move(resolved_),
                           std::move(types_), out.diagnostics.empty());
        return out;
    }

private:
    const AppGraph& g_;
    Context& ctx_;
    const KernelRegistry& reg_;
    std::vector<Diagnostic> diags_;
    std::map<ObjectId, ResolvedDesc> resolved_;
    std::map<ObjectId, std::vector<ScalarType>> types_;

    void diag(DiagCode c, std::vector<ObjectId> s, std::string m) {
        diags_.push_back(Diagnostic{c, std::move(s), std::move(m)});
    }

    const KernelSignature* signature(const OperatorNode& n, bool report) {
        if (n.abstraction) return &n.abstraction->signature;
        if (const KernelEntry* e = reg_.find(n.kernel)) return &e->signature;
        if (report) diag(DiagCode::UnknownKernel, {n.id}, "kernel '" + n.kernel + "' is not registered");
        return nullptr;
    }

    void structure() {
        std::map<ObjectId, std::vector<ObjectId>> writers;
        for (const OperatorNode& n : g_.nodes())
            for (const Binding& b : n.bindings)
                if (b.direction == Direction::Output) writers[b.object].push_back(n.id);
        for (const auto& [obj, ws] : writers)
            if (ws.size() > 1) {
                std::vector<ObjectId> s{obj};
                s.insert(s.end(), ws.begin(), ws.end());
                diag(DiagCode::MultipleWriters, std::move(s),
                     "data object has " + std::to_string(ws.size()) + " producers");
            }
        for (const OperatorNode& n : g_.nodes())
            for (const Binding& b : n.bindings) {
                if (g_.node(b.object))
                    diag(DiagCode::NotBipartite, {n.id, b.object}, "node is wired to another node");
                else if (!ctx_.find(b.object))
                    diag(DiagCode::UnboundParam, {n.id, b.object},
                         "binding targets a released or unknown object");
            }
        try {
            g_.topo_sort();
        } catch (const Error& e) {
            if (e.code() != ErrorCode::CycleDetected) throw;
            diag(DiagCode::CycleDetected, {g_.id()}, "graph contains a cycle");
        }
    }

    void params(const OperatorNode& n) {
        const KernelSignature* sig = signature(n, true);
        if (!sig) return;
        for (std::size_t i = 0; i < sig->params.size(); ++i) {
            const SignatureParam& p = sig->params[i];
            const std::string where = "parameter " + std::to_string(i);
            const Binding* b = n.binding_for(static_cast<int>(i));
            if (!b) {
                if (p.state == ParamState::Required)
                    diag(DiagCode::UnboundParam, {n.id},
                         "required " + where + " (" + p.name + ") of '" + n.kernel + "' is unbound");
                continue;
            }
            const DataObject* o = ctx_.find(b->object);
            if (!o) continue;
            if (o->kind != p.kind) {
                diag(DiagCode::DirectionMismatch, {n.id, b->object},
                     where + " of '" + n.kernel + "' expects " + to_string(p.kind) + ", got " +
                         to_string(o->kind));
                continue;
            }
            if (p.kind == ObjKind::Image && !p.formats.empty() && !o->is_virtual &&
                std::find(p.formats.begin(), p.formats.end(), o->format) == p.formats.end())
                diag(DiagCode::FormatMismatch, {n.id, b->object},
                     where + " of '" + n.kernel + "' does not accept format " + to_string(o->format));
            if (o->is_virtual && o->kind != ObjKind::Image && b->direction == Direction::Input &&
                g_.producer(b->object) == kInvalidId)
                diag(DiagCode::UnresolvedVirtualFormat, {b->object}, "virtual object consumed but never produced");
        }
        for (const Binding& b : n.bindings)
            if (b.param < 0 || b.param >= static_cast<int>(sig->params.size()))
                diag(DiagCode::DirectionMismatch, {n.id, b.object},
                     "'" + n.kernel + "' has no parameter " + std::to_string(b.param));
    }

    void assign(const OperatorNode& n, ObjectId out, const ResolvedDesc& want) {
        if (!ctx_.find(out)) return;
        auto it = resolved_.find(out);
        if (it == resolved_.end()) {
            resolved_[out] = want;
            return;
        }
        const ResolvedDesc& have = it->second;
        if (have.kind != want.kind) return;
        bool clash = false;
        switch (want.kind) {
        case ObjKind::Image:
            clash = have.width != want.width || have.height != want.height || have.format != want.format;
            break;
        case ObjKind::Scalar: clash = have.element_type != want.element_type; break;
        case ObjKind::Array:
            clash = have.element_type != want.element_type || have.capacity != want.capacity;
            break;
        case ObjKind::Matrix: break;
        }
        if (!clash) return;
        std::vector<ObjectId> s{out, n.id};
        for (ObjectId c : g_.consumers(out)) s.push_back(c);
        diag(DiagCode::FormatMismatch, std::move(s),
             "producer '" + n.kernel + "' resolves object to " + describe(want) + ", conflicting with " +
                 describe(have));
    }

    /// false = inputs not resolved yet (retry on the next sweep).
    bool infer(const OperatorNode& n) {
        const KernelEntry* entry = nullptr;
        const KernelSignature* sig = nullptr;
        if (n.abstraction) {
            sig = &n.abstraction->signature;
        } else {
            entry = reg_.find(n.kernel);
            if (!entry) return true;
            sig = &entry->signature;
        }
        std::vector<ResolvedDesc> ins;
        std::vector<ObjectId> outs;
        for (std::size_t i = 0; i < sig->params.size(); ++i) {
            const SignatureParam& p = sig->params[i];
            const Binding* b = n.binding_for(static_cast<int>(i));
            if (p.direction == Direction::Output) {
                outs.push_back(b ? b->object : kInvalidId);
                continue;
            }
            if (!b) {
                if (p.state == ParamState::Required) return true;
                ins.push_back(ResolvedDesc{});
                continue;
            }
            auto it = resolved_.find(b->object);
            if (it == resolved_.end()) return false;
            if (it->second.kind == ObjKind::Image && !image_ready(it->second)) return false;
            if (it->second.kind != p.kind) return true;
            ins.push_back(it->second);
        }
        std::vector<ResolvedDesc> result;
        try {
            InferArgs a;
            a.inputs = ins;
            a.attrs = &n.attrs;
            a.node = &n;
            a.ctx = &ctx_;
            if (n.abstraction) {
                std::vector<ScalarType> t;
                result = infer_abstraction(*n.abstraction, a, &t);
                types_[n.id] = std::move(t);
            } else {
                result = entry->infer(a);
            }
        } catch (const Error& e) {
            diag(DiagCode::FormatMismatch, {n.id}, "'" + n.kernel + "': " + e.what());
            return true;
        }
        for (std::size_t i = 0; i < result.size() && i < outs.size(); ++i)
            if (outs[i] != kInvalidId) assign(n, outs[i], result[i]);
        return true;
    }

    void propagate() {
        for (ObjectId id : g_.data()) {
            const DataObject* o = ctx_.find(id);
            if (!o) continue;
            const bool concrete =
                o->kind != ObjKind::Image || (o->format != ImageFormat::UNRESOLVED && o->width > 0);
            if (!o->is_virtual || concrete) resolved_[id] = o->desc();
        }
        std::vector<ObjectId> order;
        try {
            order = g_.topo_sort();
        } catch (const Error&) {
            return;
        }
        std::set<ObjectId> done;
        for (bool moved = true; moved;) {
            moved = false;
            for (ObjectId nid : order) {
                if (done.count(nid)) continue;
                const OperatorNode* n = g_.node(nid);
                if (n && infer(*n)) {
                    done.insert(nid);
                    moved = true;
                }
            }
        }
        for (ObjectId id : g_.data()) {
            const DataObject* o = ctx_.find(id);
            if (!o || !o->is_virtual) continue;
            auto it = resolved_.find(id);
            bool ok = it != resolved_.end();
            if (ok && o->kind == ObjKind::Image) ok = image_ready(it->second);
            if (!ok)
                diag(DiagCode::UnresolvedVirtualFormat, {id},
                     "virtual object '" + o->name + "' could not be resolved");
        }
    }
};

} // namespace

VerifyResult verify(const AppGraph& g) { return Checker(g).run(); }

} // namespace gvx
