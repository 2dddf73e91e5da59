// Verification-time optimizations (paper §5).
//   DCE (Algorithm 1)        ref:src/optimize.cpp:32-85
//   transfer planning        ref:src/optimize.cpp:89-152
//   pairwise fusion rules    ref:src/optimize.cpp:287-565
//   optimize pipeline        ref:src/optimize.cpp:571-618
// The fused graph is derived from the source graph (AppGraph::derive_from),
// so fusing across virtual images works (the reference throws
// CrossGraphVirtual there).  Fusions that would change results versus
// run_naive are refused (see optimize.hpp).
#include "graphvx/optimize.hpp"

#include <algorithm>
#include <functional>
#include <tuple>

namespace gvx {

std::vector<ObjectId> FilteredGraph::alive_nodes() const {
    std::vector<ObjectId> out;
    for (ObjectId id : base_.graph().topo_sort())
        if (is_alive(id)) out.push_back(id);
    return out;
}

std::vector<ObjectId> FilteredGraph::alive_data() const {
    std::vector<ObjectId> out;
    for (ObjectId id : base_.graph().data())
        if (is_alive(id)) out.push_back(id);
    return out;
}

std::vector<std::pair<ObjectId, ObjectId>> FilteredGraph::edges() const {
    std::vector<std::pair<ObjectId, ObjectId>> out;
    for (const auto& e : base_.graph().edges())
        if (is_alive(e.first) && is_alive(e.second)) out.push_back(e);
    return out;
}

// ---------------------------------------------------------------------- DCE

FilteredGraph eliminate_dead_nodes(const VerifiedGraph& vg) {
    if (!vg.stamped()) throw Error(ErrorCode::UnstampedGraph, "dead-computation elimination needs a stamp");
    const AppGraph& g = vg.graph();
    const Context& ctx = vg.context();

    // D_in: non-virtual sources (and pass-through data); D_out: results.
    std::set<ObjectId> sources, results;
    for (ObjectId id : g.data()) {
        const DataObject* o = ctx.find(id);
        if (!o || o->is_virtual) continue;
        const bool written = g.producer(id) != kInvalidId;
        const bool read = !g.consumers(id).empty();
        if (!written || read) sources.insert(id);
        if (written) results.insert(id);
    }

    std::map<ObjectId, std::vector<ObjectId>> preds; // transposed edges
    for (const auto& [u, v] : g.edges()) preds[v].push_back(u);
    for (auto& kv : preds) std::sort(kv.second.begin(), kv.second.end());

    std::set<ObjectId> alive, expanded;
    for (ObjectId root : results) {
        std::vector<ObjectId> stack{root};
        while (!stack.empty()) {
            ObjectId v = stack.back();
            stack.pop_back();
            alive.insert(v);
            if (v != root && sources.count(v)) continue; // stop at other inputs
            if (!expanded.insert(v).second) continue;
            auto it = preds.find(v);
            if (it != preds.end()) stack.insert(stack.end(), it->second.begin(), it->second.end());
        }
    }
    return FilteredGraph(vg, std::move(alive));
}

// ---------------------------------------------------------------- transfers

TransferPlan plan_transfers(const FilteredGraph& fg) {
    const AppGraph& g = fg.base().graph();
    const Context& ctx = fg.base().context();
    const std::vector<ObjectId> nodes = fg.alive_nodes();

    TransferPlan plan;
    plan.naive_count = static_cast<int>(nodes.size()) * 2;

    std::map<ObjectId, ObjectId> up;
    for (ObjectId n : nodes) up[n] = n;
    std::function<ObjectId(ObjectId)> root = [&](ObjectId x) {
        while (up[x] != x) x = up[x] = up[up[x]];
        return x;
    };
    auto join = [&](ObjectId a, ObjectId b) {
        a = root(a);
        b = root(b);
        if (a != b) up[std::max(a, b)] = std::min(a, b);
    };
    for (ObjectId d : fg.alive_data()) {
        const DataObject* o = ctx.find(d);
        if (!o || !o->is_virtual) continue;
        const ObjectId p = g.producer(d);
        if (p == kInvalidId || !fg.is_alive(p)) continue;
        for (ObjectId c : g.consumers(d))
            if (fg.is_alive(c)) join(p, c);
    }

    std::map<ObjectId, int> seg_of_root;
    for (ObjectId n : nodes) {
        const ObjectId r = root(n);
        auto it = seg_of_root.find(r);
        if (it == seg_of_root.end()) it = seg_of_root.emplace(r, static_cast<int>(seg_of_root.size())).first;
        plan.node_segment[n] = it->second;
    }
    plan.segment_count = static_cast<int>(seg_of_root.size());

    std::set<std::tuple<int, int, ObjectId>> moves; // (segment, 0 upload / 1 download, data)
    for (ObjectId d : fg.alive_data()) {
        const DataObject* o = ctx.find(d);
        if (!o || o->is_virtual) continue;
        const ObjectId p = g.producer(d);
        if (p != kInvalidId && fg.is_alive(p)) moves.emplace(plan.node_segment[p], 1, d);
        for (ObjectId c : g.consumers(d))
            if (fg.is_alive(c)) moves.emplace(plan.node_segment[c], 0, d);
    }
    for (const auto& [seg, dir, d] : moves)
        plan.transfers.push_back(Transfer{dir == 0 ? TransferDir::HostToDevice : TransferDir::DeviceToHost, d, seg});
    return plan;
}

// ------------------------------------------------------------------- fusion

namespace {

struct Work {
    ObjectId id = kInvalidId;
    AbstractionPtr k;
    std::vector<ObjectId> ins, outs, members;
    ObjectId provenance = kInvalidId;
    std::string label;
};

/// Rewrites slot references of a point/post body.  slot_map[k] >= 0 moves
/// slot k; -1 substitutes `subst` (per RGB channel when 3 bodies).
ExprPtr reslot(const ExprPtr& e, const std::vector<int>& slot_map, const std::vector<ExprPtr>* subst) {
    if (!e) return e;
    auto copy_with_slot = [&](int slot) {
        auto c = std::make_shared<Expr>(*e);
        c->input = slot;
        if (e->op == ExprOp::ArrayAt) c->a = reslot(e->a, slot_map, subst);
        return ExprPtr(c);
    };
    switch (e->op) {
    case ExprOp::InputPixel: {
        const int m = slot_map[static_cast<std::size_t>(e->input)];
        if (m >= 0) return copy_with_slot(m);
        std::size_t ch = 0;
        if (subst->size() == 3) ch = e->channel == Channel::G ? 1 : e->channel == Channel::B ? 2 : 0;
        return (*subst)[ch];
    }
    case ExprOp::WindowPixel:
    case ExprOp::ArrayAt: return copy_with_slot(slot_map[static_cast<std::size_t>(e->input)]);
    default: break;
    }
    if (!e->a && !e->b && !e->c) return e;
    auto c = std::make_shared<Expr>(*e);
    c->a = reslot(e->a, slot_map, subst);
    c->b = reslot(e->b, slot_map, subst);
    c->c = reslot(e->c, slot_map, subst);
    return c;
}

/// Point body evaluated at tap offset (dx, dy): image reads become windows.
ExprPtr at_tap(const ExprPtr& e, const std::vector<int>& slot_map, const std::vector<bool>& image_slot,
               int dx, int dy) {
    if (!e) return e;
    if (e->op == ExprOp::InputPixel) {
        const std::size_t k = static_cast<std::size_t>(e->input);
        if (image_slot[k]) return window_pixel(slot_map[k], dx, dy, e->channel);
        auto c = std::make_shared<Expr>(*e);
        c->input = slot_map[k];
        return c;
    }
    if (e->op == ExprOp::ArrayAt) {
        auto c = std::make_shared<Expr>(*e);
        c->input = slot_map[static_cast<std::size_t>(e->input)];
        c->a = at_tap(e->a, slot_map, image_slot, dx, dy);
        return c;
    }
    if (!e->a && !e->b && !e->c) return e;
    auto c = std::make_shared<Expr>(*e);
    c->a = at_tap(e->a, slot_map, image_slot, dx, dy);
    c->b = at_tap(e->b, slot_map, image_slot, dx, dy);
    c->c = at_tap(e->c, slot_map, image_slot, dx, dy);
    return c;
}

class Fuser {
public:
    Fuser(const FilteredGraph& fg, Context& ctx) : fg_(fg), ctx_(ctx) {}

    FusionResult run() {
        const AppGraph& g = fg_.base().graph();
        for (ObjectId nid : fg_.alive_nodes()) {
            const OperatorNode* n = g.node(nid);
            Work w;
            w.id = nid;
            w.k = n->abstraction;
            w.members = {nid};
            w.provenance = n->provenance;
            w.label = n->label.empty() ? n->kernel : n->label;
            const auto& ps = n->abstraction->signature.params;
            for (std::size_t i = 0; i < ps.size(); ++i) {
                const Binding* b = n->binding_for(static_cast<int>(i));
                (ps[i].direction == Direction::Input ? w.ins : w.outs).push_back(b ? b->object : kInvalidId);
            }
            work_.push_back(std::move(w));
        }
        while (step()) {
        }
        FusionResult res;
        AppGraph& fused = ctx_.create_graph(GraphPhase::Implementation);
        fused.derive_from(g);
        res.fused = &fused;
        for (Work& w : work_) {
            std::vector<ObjectId> args;
            std::size_t ii = 0, oi = 0;
            for (const SignatureParam& p : w.k->signature.params)
                args.push_back(p.direction == Direction::Input ? w.ins[ii++] : w.outs[oi++]);
            OperatorNode& n = fused.add_abstraction_node(w.k, args, w.provenance, w.label);
            if (w.members.size() >= 2) res.groups.push_back(FusedKernel{w.members, w.k, n.id});
        }
        return res;
    }

private:
    const FilteredGraph& fg_;
    Context& ctx_;
    std::vector<Work> work_;

    ObjKind kind(ObjectId id) const { return ctx_.at(id).kind; }

    int only_reader(ObjectId data, int skip) const {
        int found = -1;
        for (std::size_t i = 0; i < work_.size(); ++i) {
            if (static_cast<int>(i) == skip) continue;
            if (std::find(work_[i].ins.begin(), work_[i].ins.end(), data) == work_[i].ins.end()) continue;
            if (found != -1) return -1;
            found = static_cast<int>(i);
        }
        return found;
    }

    static bool single_body_point(const AbstractionKernel& k) {
        return k.point().outputs.size() == 1 && k.point().outputs[0].channel_bodies.size() == 1;
    }

    bool step() {
        for (std::size_t ui = 0; ui < work_.size(); ++ui) {
            const Work& u = work_[ui];
            const AbstractionKind uk = u.k->kind;
            if (uk != AbstractionKind::Point && uk != AbstractionKind::Local) continue;
            if (u.outs.size() != 1) continue;
            const ObjectId via = u.outs[0];
            const DataObject* o = ctx_.find(via);
            if (!o || !o->is_virtual) continue;
            const int wi = only_reader(via, static_cast<int>(ui));
            if (wi < 0) continue;
            const Work& w = work_[static_cast<std::size_t>(wi)];
            const AbstractionKind wk = w.k->kind;
            if (uk == AbstractionKind::Point && wk == AbstractionKind::Point) {
                merge_pp(ui, static_cast<std::size_t>(wi), via);
                return true;
            }
            if (uk == AbstractionKind::Local && wk == AbstractionKind::Point && w.outs.size() == 1 &&
                single_body_point(*w.k) && u.k->local().boundary != BoundaryMode::Undefined) {
                merge_lp(ui, static_cast<std::size_t>(wi), via);
                return true;
            }
            if (uk == AbstractionKind::Point && wk == AbstractionKind::Local && !w.ins.empty() &&
                w.ins[0] == via && std::count(w.ins.begin(), w.ins.end(), via) == 1 &&
                single_body_point(*u.k) && w.k->local().boundary != BoundaryMode::Constant) {
                merge_pl(ui, static_cast<std::size_t>(wi));
                return true;
            }
        }
        return false;
    }

    KernelSignature signature_for(const std::vector<ObjectId>& ins, const Work& sink) const {
        std::vector<SignatureParam> ps;
        for (ObjectId id : ins) {
            SignatureParam p;
            p.direction = Direction::Input;
            p.kind = kind(id);
            p.element_type = ctx_.at(id).element_type;
            p.name = "in" + std::to_string(ps.size());
            ps.push_back(p);
        }
        const ImageFormat out_fmt = fg_.base().resolved().count(sink.outs[0])
                                        ? fg_.base().desc(sink.outs[0]).format
                                        : ImageFormat::UNRESOLVED;
        int oi = 0;
        for (const SignatureParam& sp : sink.k->signature.params) {
            if (sp.direction != Direction::Output) continue;
            SignatureParam p = sp;
            p.name = "out" + std::to_string(oi++);
            if (p.kind == ObjKind::Image && out_fmt != ImageFormat::UNRESOLVED) p.formats = {out_fmt};
            ps.push_back(p);
        }
        return KernelSignature(std::move(ps));
    }

    void replace(std::size_t ui, std::size_t wi, AbstractionPtr k, std::vector<ObjectId> ins) {
        const Work& u = work_[ui];
        const Work& w = work_[wi];
        Work m;
        m.id = ctx_.allocate_id();
        m.k = std::move(k);
        m.ins = std::move(ins);
        m.outs = w.outs;
        m.members = u.members;
        m.members.insert(m.members.end(), w.members.begin(), w.members.end());
        m.provenance = w.provenance;
        m.label = u.label + "+" + w.label;
        const std::size_t lo = std::min(ui, wi), hi = std::max(ui, wi);
        work_.erase(work_.begin() + static_cast<std::ptrdiff_t>(hi));
        work_[lo] = std::move(m);
    }

    // point -> point: the producer body replaces every read of `via`.
    void merge_pp(std::size_t ui, std::size_t wi, ObjectId via) {
        const Work u = work_[ui];
        const Work w = work_[wi];
        std::vector<ObjectId> ins;
        std::vector<int> wmap(w.ins.size());
        for (std::size_t j = 0; j < w.ins.size(); ++j) {
            if (w.ins[j] == via) {
                wmap[j] = -1;
            } else {
                wmap[j] = static_cast<int>(ins.size());
                ins.push_back(w.ins[j]);
            }
        }
        std::vector<int> umap(u.ins.size());
        for (std::size_t i = 0; i < u.ins.size(); ++i) {
            umap[i] = static_cast<int>(ins.size());
            ins.push_back(u.ins[i]);
        }
        std::vector<ExprPtr> subst;
        for (const ExprPtr& b : u.k->point().outputs[0].channel_bodies) subst.push_back(reslot(b, umap, nullptr));
        PointKernel pk;
        pk.arity = static_cast<int>(ins.size());
        for (const PointOutput& po : w.k->point().outputs) {
            PointOutput npo;
            for (const ExprPtr& b : po.channel_bodies) npo.channel_bodies.push_back(reslot(b, wmap, &subst));
            pk.outputs.push_back(std::move(npo));
        }
        AbstractionPtr k = make_point_kernel(u.label + "+" + w.label, signature_for(ins, w), std::move(pk));
        replace(ui, wi, std::move(k), std::move(ins));
    }

    // local -> point: the point body becomes the local's post body.
    void merge_lp(std::size_t ui, std::size_t wi, ObjectId via) {
        const Work u = work_[ui];
        const Work w = work_[wi];
        const LocalKernel& ul = u.k->local();
        std::vector<ObjectId> ins = u.ins;
        std::vector<int> wmap(w.ins.size());
        for (std::size_t j = 0; j < w.ins.size(); ++j) {
            if (w.ins[j] == via) {
                wmap[j] = -1;
            } else {
                wmap[j] = static_cast<int>(ins.size());
                ins.push_back(w.ins[j]);
            }
        }
        std::vector<ExprPtr> subst{ul.post_body ? ul.post_body : input_pixel(0)};
        LocalKernel lk = ul;
        lk.post_body = reslot(w.k->point().outputs[0].channel_bodies[0], wmap, &subst);
        lk.point_arity = static_cast<int>(ins.size() - u.ins.size()) + ul.point_arity;
        AbstractionPtr k = make_local_kernel(u.label + "+" + w.label, signature_for(ins, w), std::move(lk));
        replace(ui, wi, std::move(k), std::move(ins));
    }

    // point -> local: the point body is inlined at every tap of window input 0.
    void merge_pl(std::size_t ui, std::size_t wi) {
        const Work u = work_[ui];
        const Work w = work_[wi];
        const LocalKernel& wl = w.k->local();
        std::vector<ObjectId> ins = u.ins;
        std::vector<int> umap(u.ins.size());
        std::vector<bool> uimg(u.ins.size());
        for (std::size_t i = 0; i < u.ins.size(); ++i) {
            umap[i] = static_cast<int>(i);
            uimg[i] = kind(u.ins[i]) == ObjKind::Image;
        }
        std::vector<int> wmap(w.ins.size(), -1);
        for (std::size_t j = 1; j < w.ins.size(); ++j) {
            wmap[j] = static_cast<int>(ins.size());
            ins.push_back(w.ins[j]);
        }
        const ExprPtr& body = u.k->point().outputs[0].channel_bodies[0];
        std::function<ExprPtr(const ExprPtr&)> tap = [&](const ExprPtr& e) -> ExprPtr {
            if (!e) return e;
            if (e->op == ExprOp::WindowPixel) {
                const int m = wmap[static_cast<std::size_t>(e->input)];
                if (m < 0) return at_tap(body, umap, uimg, e->dx, e->dy);
                auto c = std::make_shared<Expr>(*e);
                c->input = m;
                return c;
            }
            if (e->op == ExprOp::InputPixel || e->op == ExprOp::ArrayAt) {
                auto c = std::make_shared<Expr>(*e);
                c->input = wmap[static_cast<std::size_t>(e->input)];
                if (e->op == ExprOp::ArrayAt) c->a = tap(e->a);
                return c;
            }
            if (!e->a && !e->b && !e->c) return e;
            auto c = std::make_shared<Expr>(*e);
            c->a = tap(e->a);
            c->b = tap(e->b);
            c->c = tap(e->c);
            return c;
        };
        LocalKernel lk = wl;
        lk.tap_body = tap(wl.tap_body);
        if (wl.post_body) {
            std::vector<int> pmap(w.ins.size());
            pmap[0] = 0;
            for (std::size_t j = 1; j < w.ins.size(); ++j) pmap[j] = wmap[j];
            lk.post_body = reslot(wl.post_body, pmap, nullptr);
        }
        AbstractionPtr k = make_local_kernel(u.label + "+" + w.label, signature_for(ins, w), std::move(lk));
        replace(ui, wi, std::move(k), std::move(ins));
    }
};

} // namespace

FusionResult fuse(const FilteredGraph& g, Context& ctx) { return Fuser(g, ctx).run(); }

OptimizedPlan optimize(const VerifiedGraph& g, Context& ctx, const OptimizeOptions& opt) {
    OptimizedPlan plan;
    plan.base = g;
    plan.stats.nodes_before = static_cast<int>(g.graph().nodes().size());
    if (opt.dce) {
        plan.filtered = eliminate_dead_nodes(g);
    } else {
        std::set<ObjectId> all(g.graph().data().begin(), g.graph().data().end());
        for (const OperatorNode& n : g.graph().nodes()) all.insert(n.id);
        plan.filtered = FilteredGraph(g, std::move(all));
    }
    plan.stats.nodes_alive = static_cast<int>(plan.filtered.alive_nodes().size());
    plan.stats.nodes_removed = plan.stats.nodes_before - plan.stats.nodes_alive;
    plan.stats.launches_before = plan.stats.nodes_alive;

    plan.transfers = plan_transfers(plan.filtered);
    plan.stats.transfers_naive = plan.transfers.naive_count;
    plan.stats.transfers_optimized = plan.transfers.optimized_count();

    FusionResult fr;
    if (opt.fusion) {
        fr = fuse(plan.filtered, ctx);
    } else {
        AppGraph& copy = ctx.create_graph(GraphPhase::Implementation);
        copy.derive_from(g.graph());
        for (ObjectId nid : plan.filtered.alive_nodes()) {
            OperatorNode n = *g.graph().node(nid);
            n.id = kInvalidId;
            copy.add_node_unchecked(std::move(n));
        }
        fr.fused = &copy;
    }
    plan.groups = fr.groups;
    plan.stats.fused_groups = static_cast<int>(fr.groups.size());
    plan.stats.launches_after = static_cast<int>(fr.fused->nodes().size());

    VerifyResult vr = verify(*fr.fused);
    if (!vr.ok()) {
        std::string msg = "fused graph failed verification:";
        for (const Diagnostic& d : vr.diagnostics) msg += "\n  " + d.render();
        throw Error(ErrorCode::BadKernel, msg);
    }
    plan.fused = std::move(vr.verified);
    return plan;
}

} // namespace gvx
