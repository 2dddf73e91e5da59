// Device-group matching: recognises fusible regions of an alive
// implementation graph that map onto the hand-written sm_100a kernels, and
// static event counting of executed nodes.
//
// Unlike the reference fuser (pairwise rules, single consumer, no
// local->local, ref:src/optimize.cpp:287-334), a group here spans
// local->local chains and multi-consumer intermediates (Sobel's gx/gy feed
// three products and the magnitude) and ends in global epilogues.  A group is
// only formed when every intermediate it keeps on chip is virtual and read
// exclusively inside the group; anything observable is stored.
// Each matcher compares the abstraction bodies structurally against the
// exact trees the registry builds (ref:src/registry.cpp:456-1010) so the
// kernel's integer shortcuts are provably equal to the reference arithmetic.
#include "program.hpp"

#include <cmath>
#include <cstring>

namespace gvx::dev {

bool GraphView::is_virtual(ObjectId id) const {
    const DataObject* o = ctx->find(id);
    return o && o->is_virtual;
}

namespace {

bool same(const ExprPtr& a, const ExprPtr& b);

bool same_node(const Expr& a, const Expr& b) {
    if (a.op != b.op) return false;
    switch (a.op) {
    case ExprOp::ConstI: return a.ival == b.ival;
    case ExprOp::ConstF: return std::memcmp(&a.fval, &b.fval, sizeof(double)) == 0;
    case ExprOp::InputPixel: return a.input == b.input && a.channel == b.channel;
    case ExprOp::WindowPixel: return a.input == b.input && a.channel == b.channel && a.dx == b.dx && a.dy == b.dy;
    case ExprOp::MaskCoef: return a.dx == b.dx && a.dy == b.dy;
    case ExprOp::ArrayAt: return a.input == b.input && same(a.a, b.a);
    case ExprOp::Cast: return a.cast_to == b.cast_to && a.policy == b.policy && same(a.a, b.a);
    default: return same(a.a, b.a) && same(a.b, b.b) && same(a.c, b.c);
    }
}

bool same(const ExprPtr& a, const ExprPtr& b) {
    if (!a || !b) return !a && !b;
    return a == b || same_node(*a, *b);
}

ExprPtr in(int k) { return input_pixel(k); }
ExprPtr sat(ScalarType t, ExprPtr e) { return cast(t, CastPolicy::Saturate, std::move(e)); }
ExprPtr tap_mw() { return mul(mask_coef(0, 0), window_pixel(0, 0, 0)); }

struct NodeIO {
    const OperatorNode* n = nullptr;
    const AbstractionKernel* k = nullptr;
    std::vector<ObjectId> ins, outs;
};

NodeIO io_of(const OperatorNode* n) {
    NodeIO io;
    io.n = n;
    io.k = n->abstraction.get();
    const auto& ps = io.k->signature.params;
    for (std::size_t i = 0; i < ps.size(); ++i) {
        const Binding* b = n->binding_for(static_cast<int>(i));
        (ps[i].direction == Direction::Input ? io.ins : io.outs).push_back(b ? b->object : kInvalidId);
    }
    return io;
}

/// Integer mask of a linear local (kernel table or bound matrix).
bool int_mask(const GraphView& v, const NodeIO& io, const LocalKernel& lk, std::vector<std::int64_t>& out) {
    const std::vector<Value>* m = &lk.mask;
    if (lk.mask.empty()) {
        m = nullptr;
        for (ObjectId id : io.ins) {
            if (id == kInvalidId || v.desc(id).kind != ObjKind::Matrix) continue;
            auto it = v.matrices->find(id);
            if (it != v.matrices->end()) m = &it->second;
            break;
        }
        if (!m) return false;
    }
    if (lk.mask_is_real || static_cast<int>(m->size()) != lk.window_w * lk.window_h) return false;
    out.clear();
    for (const Value& x : *m) {
        if (x.real) return false;
        out.push_back(x.i);
    }
    return true;
}

/// Local with Clamp / Sum / mask*window taps over one U8 image.
bool linear_local(const GraphView& v, const NodeIO& io, std::vector<std::int64_t>& mask, int& ksize) {
    if (io.k->kind != AbstractionKind::Local) return false;
    const LocalKernel& lk = io.k->local();
    if (lk.window_w != lk.window_h || lk.boundary != BoundaryMode::Clamp || lk.combine != CombineMode::Sum ||
        lk.median3x3 || lk.point_arity != 0 || !same(lk.tap_body, tap_mw()))
        return false;
    if (io.outs.size() != 1 || io.outs[0] == kInvalidId || io.ins.empty() || io.ins[0] == kInvalidId) return false;
    for (std::size_t i = 1; i < io.ins.size(); ++i)
        if (io.ins[i] != kInvalidId && v.desc(io.ins[i]).kind != ObjKind::Matrix) return false;
    if (v.desc(io.ins[0]).format != ImageFormat::U8) return false;
    ksize = lk.window_w;
    return int_mask(v, io, lk, mask);
}

/// post == sat_T(in0 * (1/d)) or sat_T(in0) with round-half-away(s/d)
/// provably equal to llround(s * fl(1/d)) (d power of two, or d odd and
/// |s| < 2^50).
bool divisor_post(const ExprPtr& post, ScalarType t, std::int64_t& d) {
    if (same(post, sat(t, in(0)))) {
        d = 1;
        return true;
    }
    if (!post || post->op != ExprOp::Cast || post->cast_to != t || post->policy != CastPolicy::Saturate) return false;
    const Expr& m = *post->a;
    if (m.op != ExprOp::Mul || !same(m.a, in(0)) || m.b->op != ExprOp::ConstF) return false;
    const double c = m.b->fval;
    if (!(c > 0.0) || c > 1.0) return false;
    const double inv = std::nearbyint(1.0 / c);
    if (inv < 1 || inv > 1 << 20) return false;
    d = static_cast<std::int64_t>(inv);
    if (1.0 / static_cast<double>(d) != c) return false;
    const bool pow2 = (d & (d - 1)) == 0;
    return pow2 || (d & 1) == 1;
}

std::int64_t abs_mask_sum(const std::vector<std::int64_t>& m) {
    std::int64_t s = 0;
    for (std::int64_t x : m) s += x < 0 ? -x : x;
    return s;
}

bool is_masked3x3(const NodeIO& io, std::initializer_list<std::int64_t> mask, const ExprPtr& post) {
    if (io.k->kind != AbstractionKind::Local) return false;
    const LocalKernel& lk = io.k->local();
    if (lk.window_w != 3 || lk.window_h != 3 || lk.boundary != BoundaryMode::Clamp ||
        lk.combine != CombineMode::Sum || lk.median3x3 || lk.point_arity != 0 || lk.mask_is_real ||
        !same(lk.tap_body, tap_mw()) || !same(lk.post_body, post) || lk.mask.size() != 9)
        return false;
    std::size_t i = 0;
    for (std::int64_t m : mask) {
        const Value& v = lk.mask[i++];
        if (v.real || v.i != m) return false;
    }
    return io.ins.size() == 1 && io.outs.size() == 1 && io.ins[0] != kInvalidId && io.outs[0] != kInvalidId;
}

bool is_point_body(const NodeIO& io, int arity, const ExprPtr& body) {
    if (io.k->kind != AbstractionKind::Point) return false;
    const PointKernel& pk = io.k->point();
    if (pk.outputs.size() != 1 || pk.outputs[0].channel_bodies.size() != 1) return false;
    if (static_cast<int>(io.ins.size()) != arity || io.outs.size() != 1 || io.outs[0] == kInvalidId) return false;
    for (ObjectId id : io.ins)
        if (id == kInvalidId) return false;
    return same(pk.outputs[0].channel_bodies[0], body);
}

const ExprPtr& point_body(const NodeIO& io) { return io.k->point().outputs[0].channel_bodies[0]; }

/// Readers of `obj` among alive nodes.
const std::vector<ObjectId>& readers(const GraphView& v, ObjectId obj) {
    static const std::vector<ObjectId> none;
    auto it = v.readers.find(obj);
    return it == v.readers.end() ? none : it->second;
}

bool only_read_by(const GraphView& v, ObjectId obj, const std::set<ObjectId>& allowed) {
    if (!v.is_virtual(obj)) return false;
    for (ObjectId r : readers(v, obj))
        if (!allowed.count(r)) return false;
    return true;
}

bool is_single_reader(const GraphView& v, ObjectId obj, ObjectId reader) {
    const auto& r = readers(v, obj);
    return v.is_virtual(obj) && r.size() == 1 && r[0] == reader;
}

// --------------------------------------------------------------- edge (K1)

const std::initializer_list<std::int64_t> kSobelX = {-1, 0, 1, -2, 0, 2, -1, 0, 1};
const std::initializer_list<std::int64_t> kSobelY = {-1, -2, -1, 0, 0, 0, 1, 2, 1};
const std::initializer_list<std::int64_t> kGauss = {1, 2, 1, 2, 4, 2, 1, 2, 1};
const std::initializer_list<std::int64_t> kBox = {1, 1, 1, 1, 1, 1, 1, 1, 1};

ExprPtr sobel_post() { return sat(ScalarType::S16, in(0)); }
ExprPtr gauss_post() { return sat(ScalarType::U8, mul(in(0), const_f(1.0 / 16.0))); }
ExprPtr magnitude_body() {
    return sat(ScalarType::S16, unary(ExprOp::Sqrt, add(mul(in(0), in(0)), mul(in(1), in(1)))));
}

void match_edges(const GraphView& v, std::set<ObjectId>& used, std::vector<Unit>& out) {
    std::map<ObjectId, std::pair<const OperatorNode*, const OperatorNode*>> by_src; // src -> (sx, sy)
    for (const OperatorNode* n : v.nodes) {
        if (used.count(n->id)) continue;
        NodeIO io = io_of(n);
        if (is_masked3x3(io, kSobelX, sobel_post()) && v.desc(io.ins[0]).format == ImageFormat::U8)
            by_src[io.ins[0]].first = n;
        else if (is_masked3x3(io, kSobelY, sobel_post()) && v.desc(io.ins[0]).format == ImageFormat::U8)
            by_src[io.ins[0]].second = n;
    }
    for (auto& [src, pair] : by_src) {
        const OperatorNode* sx = pair.first;
        const OperatorNode* sy = pair.second;
        Unit u;
        u.kind = Unit::Kind::Edge;
        u.label = "edge";
        ObjectId gx = sx ? io_of(sx).outs[0] : kInvalidId;
        ObjectId gy = sy ? io_of(sy).outs[0] : kInvalidId;
        std::set<ObjectId> group;
        if (sx) group.insert(sx->id);
        if (sy) group.insert(sy->id);
        // magnitude over (gx, gy)
        const OperatorNode* mag = nullptr;
        if (sx && sy)
            for (ObjectId r : readers(v, gx)) {
                const OperatorNode* n = v.vg->graph().node(r);
                if (used.count(r)) continue;
                NodeIO io = io_of(n);
                if (is_point_body(io, 2, magnitude_body()) && io.ins[0] == gx && io.ins[1] == gy) {
                    mag = n;
                    break;
                }
            }
        if (mag) group.insert(mag->id);
        // store gx / gy unless they are virtual and read only by the magnitude
        auto keep = [&](ObjectId id) {
            if (id == kInvalidId) return false;
            if (!v.is_virtual(id)) return true;
            for (ObjectId r : readers(v, id))
                if (!group.count(r)) return true;
            return false;
        };
        u.out[0] = keep(gx) ? gx : kInvalidId;
        u.out[1] = keep(gy) ? gy : kInvalidId;
        u.out[2] = mag ? io_of(mag).outs[0] : kInvalidId;
        if (u.out[0] == kInvalidId && u.out[1] == kInvalidId && u.out[2] == kInvalidId) continue;
        // fuse the Gaussian that produces a virtual source read only by these Sobels
        u.src = src;
        auto w = v.writer.find(src);
        if (w != v.writer.end() && !used.count(w->second)) {
            const OperatorNode* g = v.vg->graph().node(w->second);
            NodeIO gio = io_of(g);
            if (is_masked3x3(gio, kGauss, gauss_post()) && v.desc(gio.ins[0]).format == ImageFormat::U8 &&
                only_read_by(v, src, group)) {
                u.with_gauss = true;
                u.src = gio.ins[0];
                group.insert(g->id);
            }
        }
        u.covers.assign(group.begin(), group.end());
        u.reads = {u.src};
        for (ObjectId o : u.out)
            if (o != kInvalidId) u.writes.push_back(o);
        used.insert(group.begin(), group.end());
        out.push_back(std::move(u));
    }
}

// ------------------------------------------------------------- harris (K2)

ExprPtr product_body() { return sat(ScalarType::S32, mul(in(0), in(1))); }
ExprPtr box_s32_post() { return sat(ScalarType::S32, mul(in(0), const_f(1.0 / 9.0))); }

/// F32((a*b - c*c) - k*((a+b)*(a+b))) with {a,b} = {xx,yy}, c = xy.
bool harris_response(const ExprPtr& body, int& sa, int& sb, int& sc, double& k) {
    if (!body || body->op != ExprOp::Cast || body->cast_to != ScalarType::F32 ||
        body->policy != CastPolicy::Saturate)
        return false;
    const Expr& r = *body->a;
    if (r.op != ExprOp::Sub) return false;
    const Expr& det = *r.a;
    const Expr& kt = *r.b;
    if (det.op != ExprOp::Sub || det.a->op != ExprOp::Mul || det.b->op != ExprOp::Mul) return false;
    auto slot = [](const ExprPtr& e) { return e->op == ExprOp::InputPixel && e->channel == Channel::C0 ? e->input : -1; };
    sa = slot(det.a->a);
    sb = slot(det.a->b);
    sc = slot(det.b->a);
    if (sa < 0 || sb < 0 || sc < 0 || slot(det.b->b) != sc || sa == sb || sa == sc || sb == sc) return false;
    if (kt.op != ExprOp::Mul || kt.a->op != ExprOp::ConstF || kt.b->op != ExprOp::Mul) return false;
    k = kt.a->fval;
    const ExprPtr tr = add(in(sa), in(sb));
    const ExprPtr tr2 = add(in(sb), in(sa));
    return (same(kt.b->a, tr) || same(kt.b->a, tr2)) && (same(kt.b->b, tr) || same(kt.b->b, tr2));
}

bool threshold_f32(const ExprPtr& body, double& t) {
    if (!body || body->op != ExprOp::Cast || body->cast_to != ScalarType::U8 || body->policy != CastPolicy::Saturate)
        return false;
    const Expr& s = *body->a;
    if (s.op != ExprOp::Select || s.a->op != ExprOp::Gt || !same(s.a->a, in(0)) || s.a->b->op != ExprOp::ConstF)
        return false;
    t = s.a->b->fval;
    return same(s.b, const_i(255)) && same(s.c, const_i(0));
}

void match_harris(const GraphView& v, std::set<ObjectId>& used, std::vector<Unit>& out) {
    std::map<ObjectId, std::pair<const OperatorNode*, const OperatorNode*>> by_src;
    for (const OperatorNode* n : v.nodes) {
        if (used.count(n->id)) continue;
        NodeIO io = io_of(n);
        if (is_masked3x3(io, kSobelX, sobel_post()) && v.desc(io.ins[0]).format == ImageFormat::U8)
            by_src[io.ins[0]].first = n;
        else if (is_masked3x3(io, kSobelY, sobel_post()) && v.desc(io.ins[0]).format == ImageFormat::U8)
            by_src[io.ins[0]].second = n;
    }
    for (auto& [src, pair] : by_src) {
        if (!pair.first || !pair.second) continue;
        const ObjectId gx = io_of(pair.first).outs[0], gy = io_of(pair.second).outs[0];
        if (!v.is_virtual(gx) || !v.is_virtual(gy)) continue;
        // three products
        const OperatorNode *pxx = nullptr, *pyy = nullptr, *pxy = nullptr;
        bool bad = false;
        std::set<ObjectId> prod_nodes;
        for (ObjectId r : readers(v, gx)) prod_nodes.insert(r);
        for (ObjectId r : readers(v, gy)) prod_nodes.insert(r);
        for (ObjectId r : prod_nodes) {
            const OperatorNode* n = v.vg->graph().node(r);
            NodeIO io = io_of(n);
            if (used.count(r) || !is_point_body(io, 2, product_body())) {
                bad = true;
                break;
            }
            const ObjectId a = io.ins[0], b = io.ins[1];
            if (a == gx && b == gx) pxx = n;
            else if (a == gy && b == gy) pyy = n;
            else if ((a == gx && b == gy) || (a == gy && b == gx)) pxy = n;
            else bad = true;
        }
        if (bad || !pxx || !pyy || !pxy || prod_nodes.size() != 3) continue;
        // three boxes, each the only reader of its product
        const OperatorNode* boxes[3] = {nullptr, nullptr, nullptr};
        const OperatorNode* prods[3] = {pxx, pyy, pxy};
        for (int i = 0; i < 3 && !bad; ++i) {
            const ObjectId p = io_of(prods[i]).outs[0];
            const auto& rs = readers(v, p);
            if (!v.is_virtual(p) || rs.size() != 1 || used.count(rs[0])) {
                bad = true;
                break;
            }
            const OperatorNode* b = v.vg->graph().node(rs[0]);
            NodeIO bio = io_of(b);
            if (!is_masked3x3(bio, kBox, box_s32_post()) || v.desc(bio.outs[0]).format != ImageFormat::S32) bad = true;
            boxes[i] = b;
        }
        if (bad) continue;
        const ObjectId sxx = io_of(boxes[0]).outs[0], syy = io_of(boxes[1]).outs[0], sxy = io_of(boxes[2]).outs[0];
        // response point node reading the three box outputs
        const auto& rr = readers(v, sxx);
        if (!v.is_virtual(sxx) || !v.is_virtual(syy) || !v.is_virtual(sxy) || rr.size() != 1) continue;
        const OperatorNode* resp = v.vg->graph().node(rr[0]);
        NodeIO rio = io_of(resp);
        if (used.count(resp->id) || rio.k->kind != AbstractionKind::Point || rio.ins.size() != 3 ||
            !is_point_body(rio, 3, point_body(rio)))
            continue;
        if (readers(v, syy) != rr || readers(v, sxy) != rr) continue;
        int sa, sb, sc;
        double kk;
        if (!harris_response(point_body(rio), sa, sb, sc, kk)) continue;
        const ObjectId A = rio.ins[static_cast<std::size_t>(sa)], B = rio.ins[static_cast<std::size_t>(sb)],
                       C = rio.ins[static_cast<std::size_t>(sc)];
        if (C != sxy || !((A == sxx && B == syy) || (A == syy && B == sxx))) continue;
        const ObjectId respo = rio.outs[0];
        if (v.desc(respo).format != ImageFormat::F32) continue;
        // threshold point node
        const auto& tr = readers(v, respo);
        if (tr.size() != 1 || used.count(tr[0])) continue;
        const OperatorNode* thr = v.vg->graph().node(tr[0]);
        NodeIO tio = io_of(thr);
        double T;
        if (tio.k->kind != AbstractionKind::Point || !is_point_body(tio, 1, point_body(tio)) ||
            !threshold_f32(point_body(tio), T) || v.desc(tio.outs[0]).format != ImageFormat::U8)
            continue;
        Unit u;
        u.kind = Unit::Kind::Harris;
        u.label = "harris";
        u.src = src;
        u.out[0] = tio.outs[0];
        u.out[1] = v.is_virtual(respo) ? kInvalidId : respo;
        u.k_param = kk;
        u.threshold = T;
        u.covers = {pair.first->id, pair.second->id, pxx->id, pyy->id, pxy->id, boxes[0]->id, boxes[1]->id,
                    boxes[2]->id, resp->id, thr->id};
        u.reads = {src};
        u.writes = {u.out[0]};
        if (u.out[1] != kInvalidId) u.writes.push_back(u.out[1]);
        used.insert(u.covers.begin(), u.covers.end());
        out.push_back(std::move(u));
    }
}

// ------------------------------------------- linear stencil + points (K3)

void match_stencils(const GraphView& v, std::set<ObjectId>& used, std::vector<Unit>& out) {
    static const bool off = std::getenv("GVX_NO_K3") != nullptr; // A/B: leave linear stencils to the generic path
    if (off) return;
    for (const OperatorNode* n : v.nodes) {
        if (used.count(n->id)) continue;
        NodeIO io = io_of(n);
        std::vector<std::int64_t> mask;
        int ks = 0;
        if (!linear_local(v, io, mask, ks) || (ks != 3 && ks != 5 && ks != 7)) continue;
        const ObjectId src = io.ins[0], blur = io.outs[0];
        if (v.desc(blur).format != ImageFormat::U8) continue;
        std::int64_t d = 1;
        if (!divisor_post(io.k->local().post_body, ScalarType::U8, d)) continue;
        if (abs_mask_sum(mask) * 255 >= (1ll << 30)) continue;
        Unit u;
        u.kind = Unit::Kind::Stencil;
        u.label = "stencil";
        u.src = src;
        u.ksize = ks;
        for (std::size_t i = 0; i < mask.size(); ++i) u.mask[i] = static_cast<int>(mask[i]);
        u.divisor = d;
        u.mode = 0;
        u.out[0] = blur;
        u.covers = {n->id};
        // unsharp chain: Subtract(src, blur) -> Add(src, diff) -> ConvertDepth(-> U8)
        if (is_single_reader(v, blur, v.readers.count(blur) ? v.readers.at(blur)[0] : kInvalidId)) {
            const OperatorNode* s = v.vg->graph().node(v.readers.at(blur)[0]);
            NodeIO sio = io_of(s);
            if (!used.count(s->id) && is_point_body(sio, 2, sat(ScalarType::S16, sub(in(0), in(1)))) &&
                sio.ins[0] == src && sio.ins[1] == blur && v.desc(sio.outs[0]).format == ImageFormat::S16) {
                const ObjectId diff = sio.outs[0];
                const auto& ar = readers(v, diff);
                if (v.is_virtual(diff) && ar.size() == 1 && !used.count(ar[0])) {
                    const OperatorNode* a = v.vg->graph().node(ar[0]);
                    NodeIO aio = io_of(a);
                    const bool add_ok =
                        is_point_body(aio, 2, sat(ScalarType::S16, add(in(0), in(1)))) &&
                        ((aio.ins[0] == src && aio.ins[1] == diff) || (aio.ins[0] == diff && aio.ins[1] == src)) &&
                        v.desc(aio.outs[0]).format == ImageFormat::S16;
                    if (add_ok) {
                        const ObjectId sum = aio.outs[0];
                        const auto& cr = readers(v, sum);
                        if (v.is_virtual(sum) && cr.size() == 1 && !used.count(cr[0])) {
                            const OperatorNode* c = v.vg->graph().node(cr[0]);
                            NodeIO cio = io_of(c);
                            if (is_point_body(cio, 1, sat(ScalarType::U8, in(0))) &&
                                v.desc(cio.outs[0]).format == ImageFormat::U8) {
                                u.mode = 1;
                                u.out[0] = cio.outs[0];
                                u.covers = {n->id, s->id, a->id, c->id};
                            }
                        }
                    }
                }
            }
        }
        if (u.mode == 0 && v.is_virtual(blur)) {
            // a lone virtual blur must still be materialised for its readers
        }
        u.reads = {src};
        u.writes = {u.out[0]};
        used.insert(u.covers.begin(), u.covers.end());
        out.push_back(std::move(u));
    }
}

// ------------------------------------ convolve -> convert -> stats (K4)

bool is_hist_standard(const NodeIO& io, int& bins, std::int64_t& off, std::int64_t& range) {
    if (io.k->kind != AbstractionKind::Histogram) return false;
    const HistogramKernel& hk = io.k->histogram();
    const ExprPtr want = div(mul(sub(in(0), const_i(hk.offset)), const_i(hk.bins)), const_i(hk.range));
    if (!same(hk.bin_of, want) || hk.range == 0) return false;
    bins = hk.bins;
    off = hk.offset;
    range = hk.range;
    return io.outs.size() == 1 && io.outs[0] != kInvalidId && bins <= 4096;
}

bool is_reduce_mean(const NodeIO& io) {
    if (io.k->kind != AbstractionKind::Reduce) return false;
    const ReduceKernel& rk = io.k->reduce();
    return !rk.seed_first && !rk.init.real && rk.init.i == 0 && rk.track == ReduceKernel::Track::None &&
           same(rk.combine, add(in(0), in(1))) &&
           same(rk.finalize, sat(ScalarType::F32, div(mul(in(0), const_f(1.0)), in(1)))) && io.ins.size() == 1 &&
           io.outs.size() == 1 && io.outs[0] != kInvalidId;
}

bool is_reduce_stddev(const NodeIO& io) {
    if (io.k->kind != AbstractionKind::Reduce) return false;
    const ReduceKernel& rk = io.k->reduce();
    const ExprPtr var = binary(ExprOp::Max, sub(div(mul(in(0), const_f(1.0)), in(1)), mul(in(2), in(2))), const_f(0.0));
    return !rk.seed_first && !rk.init.real && rk.init.i == 0 && rk.track == ReduceKernel::Track::None &&
           same(rk.combine, add(in(0), mul(in(1), in(1)))) &&
           same(rk.finalize, sat(ScalarType::F32, unary(ExprOp::Sqrt, var))) && io.ins.size() == 2 &&
           io.outs.size() == 1 && io.outs[0] != kInvalidId;
}

void match_conv_stats(const GraphView& v, std::set<ObjectId>& used, std::vector<Unit>& out) {
    for (const OperatorNode* n : v.nodes) {
        if (used.count(n->id)) continue;
        NodeIO io = io_of(n);
        std::vector<std::int64_t> mask;
        int ks = 0;
        if (!linear_local(v, io, mask, ks) || (ks != 3 && ks != 5 && ks != 7)) continue;
        const ObjectId conv = io.outs[0];
        const ImageFormat cf = v.desc(conv).format;
        if (cf != ImageFormat::S16 && cf != ImageFormat::U8) continue;
        std::int64_t d = 1;
        if (!divisor_post(io.k->local().post_body, scalar_of(cf), d)) continue;
        if (abs_mask_sum(mask) * 255 >= (1ll << 30)) continue;
        const auto& cr = readers(v, conv);
        if (!v.is_virtual(conv) || cr.size() != 1 || used.count(cr[0])) continue;
        const OperatorNode* cd = v.vg->graph().node(cr[0]);
        NodeIO cio = io_of(cd);
        if (cio.k->kind != AbstractionKind::Point || !is_point_body(cio, 1, point_body(cio))) continue;
        const ExprPtr& cb = point_body(cio);
        if (cb->op != ExprOp::Cast || cb->cast_to != ScalarType::U8) continue;
        int shift = 0;
        if (!same(cb->a, in(0))) {
            if (cb->a->op != ExprOp::Shr || !same(cb->a->a, in(0)) || cb->a->b->op != ExprOp::ConstI) continue;
            const std::int64_t s = cb->a->b->ival;
            if (s < 0 || s > 31) continue;
            shift = static_cast<int>(s);
        }
        const ObjectId u8 = cio.outs[0];
        if (v.desc(u8).format != ImageFormat::U8) continue;
        const OperatorNode *hist = nullptr, *mean = nullptr, *sd = nullptr;
        int bins = 0;
        std::int64_t off = 0, range = 0;
        bool bad = false;
        for (ObjectId r : readers(v, u8)) {
            const OperatorNode* m = v.vg->graph().node(r);
            NodeIO mio = io_of(m);
            if (used.count(r)) {
                bad = true;
            } else if (!hist && is_hist_standard(mio, bins, off, range)) {
                hist = m;
            } else if (!mean && is_reduce_mean(mio)) {
                mean = m;
            } else if (!sd && is_reduce_stddev(mio)) {
                sd = m;
            } else {
                bad = true;
            }
        }
        if (bad || (!hist && !mean)) continue;
        if (sd && (!mean || io_of(sd).ins[1] != io_of(mean).outs[0])) continue;
        Unit u;
        u.kind = Unit::Kind::ConvStats;
        u.label = "conv_stats";
        u.src = io.ins[0];
        u.ksize = ks;
        for (std::size_t i = 0; i < mask.size(); ++i) u.mask[i] = static_cast<int>(mask[i]);
        u.divisor = d;
        u.conv_format = static_cast<int>(cf);
        u.shift = shift;
        u.wrap = cb->policy == CastPolicy::Wrap ? 1 : 0;
        u.bins = hist ? bins : 1;
        u.offset = off;
        u.range = hist ? range : 1;
        u.out[0] = v.is_virtual(u8) ? kInvalidId : u8;
        u.out[1] = hist ? io_of(hist).outs[0] : kInvalidId;
        u.out[2] = mean ? io_of(mean).outs[0] : kInvalidId;
        u.out[3] = sd ? io_of(sd).outs[0] : kInvalidId;
        u.covers = {n->id, cd->id};
        for (const OperatorNode* m : {hist, mean, sd})
            if (m) u.covers.push_back(m->id);
        u.reads = {u.src};
        for (ObjectId o : u.out)
            if (o != kInvalidId) u.writes.push_back(o);
        used.insert(u.covers.begin(), u.covers.end());
        out.push_back(std::move(u));
    }
}

// ------------------------------------------------------------- counting

struct ReadTally {
    int image_reads = 0;
    bool conditional = false;
};

void tally(const Expr& e, const std::vector<bool>& image_slot, ReadTally& t, bool in_branch, int slot_shift = 0) {
    if (e.op == ExprOp::InputPixel) {
        const int s = e.input - slot_shift;
        if (s >= 0 && s < static_cast<int>(image_slot.size()) && image_slot[static_cast<std::size_t>(s)]) {
            ++t.image_reads;
            if (in_branch) t.conditional = true;
        }
        return;
    }
    if (e.op == ExprOp::WindowPixel) {
        ++t.image_reads;
        if (in_branch) t.conditional = true;
        return;
    }
    if (e.a) tally(*e.a, image_slot, t, in_branch, slot_shift);
    if (e.b) tally(*e.b, image_slot, t, in_branch || e.op == ExprOp::Select, slot_shift);
    if (e.c) tally(*e.c, image_slot, t, in_branch || e.op == ExprOp::Select, slot_shift);
}

} // namespace

std::vector<Unit> match_fused_groups(const GraphView& view) {
    std::vector<Unit> units;
    std::set<ObjectId> used;
    match_harris(view, used, units);
    match_edges(view, used, units);
    match_conv_stats(view, used, units);
    match_stencils(view, used, units);
    return units;
}

bool static_counts(const OperatorNode& n, const VerifiedGraph& vg, std::int64_t& reads, std::int64_t& writes) {
    const AbstractionKernel& k = *n.abstraction;
    NodeIO io = io_of(&n);
    std::vector<bool> image_slot;
    const ResolvedDesc* img = nullptr;
    for (ObjectId id : io.ins) {
        const bool is_img = id != kInvalidId && vg.desc(id).kind == ObjKind::Image;
        image_slot.push_back(is_img);
        if (is_img && !img) img = &vg.desc(id);
    }
    reads = writes = 0;
    switch (k.kind) {
    case AbstractionKind::Point: {
        const ResolvedDesc& d = img ? *img : vg.desc(io.outs.at(0));
        const std::int64_t px = static_cast<std::int64_t>(d.width) * d.height;
        ReadTally t;
        int slots = 0;
        for (std::size_t o = 0; o < k.point().outputs.size() && o < io.outs.size(); ++o) {
            if (io.outs[o] == kInvalidId) continue;
            ++slots;
            const auto& bodies = k.point().outputs[o].channel_bodies;
            const bool rgb = bodies.size() == 3 && vg.desc(io.outs[o]).format == ImageFormat::RGB;
            for (std::size_t c = 0; c < (rgb ? 3u : 1u); ++c) tally(*bodies[c], image_slot, t, false);
        }
        writes = px * slots; // writes are static even when reads depend on data
        if (t.conditional) return false;
        reads = px * t.image_reads;
        return true;
    }
    case AbstractionKind::Local: {
        const LocalKernel& lk = k.local();
        const ResolvedDesc& od = vg.desc(io.outs.at(0));
        const std::int64_t W = od.width, H = od.height;
        const int hw = lk.window_w / 2, hh = lk.window_h / 2;
        writes = W * H;
        std::int64_t interior = W * H;
        if (lk.boundary == BoundaryMode::Undefined)
            interior = std::max<std::int64_t>(0, W - 2 * hw) * std::max<std::int64_t>(0, H - 2 * hh);
        // tap body: pointwise image reads + window reads per tap
        ReadTally pt;
        std::vector<std::pair<int, int>> wins; // window read offsets
        std::function<void(const Expr&, bool)> walk = [&](const Expr& e, bool br) {
            if (e.op == ExprOp::WindowPixel) {
                wins.emplace_back(e.dx, e.dy);
                if (br) pt.conditional = true;
                return;
            }
            if (e.op == ExprOp::InputPixel) {
                const int s = e.input;
                if (s >= 0 && s < static_cast<int>(image_slot.size()) && image_slot[static_cast<std::size_t>(s)]) {
                    ++pt.image_reads;
                    if (br) pt.conditional = true;
                }
                return;
            }
            if (e.a) walk(*e.a, br);
            if (e.b) walk(*e.b, br || e.op == ExprOp::Select);
            if (e.c) walk(*e.c, br || e.op == ExprOp::Select);
        };
        walk(*lk.tap_body, false);
        if (pt.conditional) return false;
        const std::int64_t taps = static_cast<std::int64_t>(lk.window_w) * lk.window_h;
        reads = interior * taps * pt.image_reads;
        for (int ty = -hh; ty <= hh; ++ty)
            for (int tx = -hw; tx <= hw; ++tx)
                for (auto [dx, dy] : wins) {
                    if (lk.boundary == BoundaryMode::Constant) {
                        const std::int64_t ox = std::abs(tx + dx), oy = std::abs(ty + dy);
                        reads += std::max<std::int64_t>(0, W - ox) * std::max<std::int64_t>(0, H - oy);
                    } else {
                        reads += interior;
                    }
                }
        if (lk.post_body) {
            std::vector<bool> post_slots = image_slot;
            if (!post_slots.empty()) post_slots[0] = false; // slot 0 = combined value
            ReadTally t;
            tally(*lk.post_body, post_slots, t, false);
            if (t.conditional) return false;
            reads += interior * t.image_reads;
        }
        return true;
    }
    case AbstractionKind::Reduce: {
        const ResolvedDesc& d = vg.desc(io.ins.at(0));
        reads = static_cast<std::int64_t>(d.width) * d.height;
        writes = 1;
        if (io.outs.size() > 1 && io.outs[1] != kInvalidId && k.reduce().track != ReduceKernel::Track::None) ++writes;
        return true;
    }
    case AbstractionKind::Histogram: {
        const ResolvedDesc& d = vg.desc(io.ins.at(0));
        ReadTally t;
        tally(*k.histogram().bin_of, image_slot, t, false);
        if (t.conditional) return false;
        reads = static_cast<std::int64_t>(d.width) * d.height * t.image_reads;
        writes = k.histogram().bins;
        return true;
    }
    case AbstractionKind::Scan: {
        const ResolvedDesc& d = vg.desc(io.ins.at(0));
        reads = writes = static_cast<std::int64_t>(d.width) * d.height;
        return true;
    }
    case AbstractionKind::Scale: {
        const ResolvedDesc& d = vg.desc(io.outs.at(0));
        writes = static_cast<std::int64_t>(d.width) * d.height;
        reads = writes * (k.scale().interp == InterpMode::Nearest ? 1 : 4);
        return true;
    }
    case AbstractionKind::Table: {
        const ResolvedDesc& d = vg.desc(io.ins.at(0));
        writes = d.capacity;
        return true;
    }
    }
    return false;
}

} // namespace gvx::dev
