// CV-function catalog: OpenVX functions as compositions of point / local /
// global abstractions (paper §4), plus user-defined kernel registration and
// graph expansion.
//
// Each builtin reproduces the reference's abstraction bodies exactly (the
// expression trees decide the arithmetic, so they must match to be bit-exact):
//   signatures / default formats   ref:src/registry.cpp:14-203
//   infer_abstraction              ref:src/registry.cpp:278-337
//   add_custom                     ref:src/registry.cpp:357-376
//   pointwise builtins             ref:src/registry.cpp:402-699
//   local builtins                 ref:src/registry.cpp:701-878
//   global builtins                ref:src/registry.cpp:880-1113
//   expand                         ref:src/registry.cpp:1125-1167
// Fix vs reference: ScaleImage's abstraction declares its output format
// (= input format); the reference leaves it unconstrained and every
// ScaleImage graph fails typecheck with MissingCast (SURVEY.md §0 finding 2).
#include "graphvx/registry.hpp"
#include "graphvx/verify.hpp"

#include <algorithm>
#include <cmath>

namespace gvx {

namespace {

constexpr double kTau = 6.283185307179586476925286766559;

// ---- signature parameters --------------------------------------------------

SignatureParam param(Direction dir, ObjKind kind, std::string name,
                     std::vector<ImageFormat> fmts = {}, ScalarType et = ScalarType::F64,
                     ParamState st = ParamState::Required) {
    SignatureParam p;
    p.direction = dir;
    p.kind = kind;
    p.formats = std::move(fmts);
    p.element_type = et;
    p.state = st;
    p.name = std::move(name);
    return p;
}
SignatureParam image_in(std::string n, std::vector<ImageFormat> f = {}) {
    return param(Direction::Input, ObjKind::Image, std::move(n), std::move(f));
}
SignatureParam image_out(std::string n, std::vector<ImageFormat> f = {},
                         ParamState st = ParamState::Required) {
    return param(Direction::Output, ObjKind::Image, std::move(n), std::move(f), ScalarType::F64, st);
}

const std::vector<ImageFormat>& single_channel() {
    static const std::vector<ImageFormat> v = {ImageFormat::U8, ImageFormat::U16, ImageFormat::S16,
                                               ImageFormat::S32, ImageFormat::F32};
    return v;
}
const std::vector<ImageFormat>& integer_channel() {
    static const std::vector<ImageFormat> v = {ImageFormat::U8, ImageFormat::U16, ImageFormat::S16,
                                               ImageFormat::S32};
    return v;
}

// ---- attributes ----------------------------------------------------------------

std::int64_t get_int(const AttrMap& a, const std::string& k, std::int64_t dflt) {
    auto it = a.find(k);
    if (it == a.end()) return dflt;
    if (auto* i = std::get_if<std::int64_t>(&it->second)) return *i;
    if (auto* d = std::get_if<double>(&it->second)) return static_cast<std::int64_t>(*d);
    throw Error(ErrorCode::SchemaError, "attribute '" + k + "' must be numeric");
}
double get_real(const AttrMap& a, const std::string& k, double dflt) {
    auto it = a.find(k);
    if (it == a.end()) return dflt;
    if (auto* d = std::get_if<double>(&it->second)) return *d;
    if (auto* i = std::get_if<std::int64_t>(&it->second)) return static_cast<double>(*i);
    throw Error(ErrorCode::SchemaError, "attribute '" + k + "' must be numeric");
}
std::string get_str(const AttrMap& a, const std::string& k, const std::string& dflt) {
    auto it = a.find(k);
    if (it == a.end()) return dflt;
    if (auto* s = std::get_if<std::string>(&it->second)) return *s;
    throw Error(ErrorCode::SchemaError, "attribute '" + k + "' must be a string");
}
ImageFormat get_format(const AttrMap& a, const std::string& k, ImageFormat dflt) {
    const std::string s = get_str(a, k, "");
    if (s.empty()) return dflt;
    ImageFormat f;
    if (!parse_image_format(s, f) || f == ImageFormat::UNRESOLVED)
        throw Error(ErrorCode::BadFormat, "bad format attribute '" + s + "'");
    return f;
}
Channel get_channel(const AttrMap& a) {
    const std::string s = get_str(a, "channel", "Y");
    Channel c;
    if (!parse_channel(s, c)) throw Error(ErrorCode::SchemaError, "bad channel attribute '" + s + "'");
    return c;
}

// ---- formats ---------------------------------------------------------------------

int arith_rank(ImageFormat f) {
    switch (f) {
    case ImageFormat::U8: return 0;
    case ImageFormat::U16:
    case ImageFormat::S16: return 1;
    case ImageFormat::S32: return 2;
    case ImageFormat::F32: return 3;
    default: throw Error(ErrorCode::BadFormat, "arithmetic needs single-channel input");
    }
}
/// Sums widen one step: U8+U8 -> S16, anything with U16/S32 -> S32, F32 -> F32.
ImageFormat sum_result(ImageFormat a, ImageFormat b) {
    const int r = std::max(arith_rank(a), arith_rank(b));
    if (r == 3) return ImageFormat::F32;
    if (r == 2 || a == ImageFormat::U16 || b == ImageFormat::U16) return ImageFormat::S32;
    return ImageFormat::S16;
}
/// Products go to S32 (F32 stays F32).
ImageFormat product_result(ImageFormat a, ImageFormat b) {
    return std::max(arith_rank(a), arith_rank(b)) == 3 ? ImageFormat::F32 : ImageFormat::S32;
}

ResolvedDesc img_desc(int w, int h, ImageFormat f) {
    ResolvedDesc d;
    d.kind = ObjKind::Image;
    d.width = w;
    d.height = h;
    d.format = f;
    return d;
}
ResolvedDesc scalar_desc(ScalarType t) {
    ResolvedDesc d;
    d.kind = ObjKind::Scalar;
    d.element_type = t;
    return d;
}
ResolvedDesc array_desc(ScalarType t, std::int64_t cap) {
    ResolvedDesc d;
    d.kind = ObjKind::Array;
    d.element_type = t;
    d.capacity = cap;
    return d;
}
std::vector<ResolvedDesc> like_input(const InferArgs& a, ImageFormat f) {
    return {img_desc(a.inputs[0].width, a.inputs[0].height, f)};
}

void same_dims(const std::vector<ResolvedDesc>& in) {
    const ResolvedDesc* ref = nullptr;
    for (const ResolvedDesc& d : in) {
        if (d.kind != ObjKind::Image) continue;
        if (!ref) ref = &d;
        else if (d.width != ref->width || d.height != ref->height)
            throw Error(ErrorCode::ShapeMismatch, "input image dimensions differ");
    }
}

void scalar_within(const Context& ctx, const OperatorNode& n, int param_index, ImageFormat fmt) {
    const Binding* b = n.binding_for(param_index);
    if (!b) return;
    const DataObject* o = ctx.find(b->object);
    if (!o || !o->scalar_value) return;
    std::int64_t lo, hi;
    if (!integer_range(scalar_of(fmt), lo, hi)) return;
    const double x = o->scalar_value->as_real();
    if (x < static_cast<double>(lo) || x > static_cast<double>(hi))
        throw Error(ErrorCode::BadFormat,
                    "scalar value " + std::to_string(x) + " outside the " + to_string(fmt) + " range");
}

// ---- emission helpers -----------------------------------------------------------

ExprPtr px(int k) { return input_pixel(k); }

/// Single-output point node (inputs..., out).
void point_node(ExpandArgs& a, const std::string& label, ImageFormat out_fmt, ExprPtr body,
                const std::vector<ObjectId>& ins, ObjectId out,
                const std::vector<ObjKind>& kinds = {}) {
    std::vector<SignatureParam> ps;
    for (std::size_t i = 0; i < ins.size(); ++i)
        ps.push_back(param(Direction::Input, i < kinds.size() ? kinds[i] : ObjKind::Image,
                           "in" + std::to_string(i)));
    ps.push_back(image_out("out", {out_fmt}));
    PointKernel pk;
    pk.arity = static_cast<int>(ins.size());
    pk.outputs.push_back(PointOutput{{std::move(body)}});
    std::vector<ObjectId> args = ins;
    args.push_back(out);
    a.impl->add_abstraction_node(make_point_kernel(label, KernelSignature(std::move(ps)), std::move(pk)),
                                 args, a.node->id, label);
}

/// Single-output local node (in, [matrix], out).
void local_node(ExpandArgs& a, const std::string& label, ImageFormat out_fmt, LocalKernel lk,
                const std::vector<ObjectId>& ins, ObjectId out, bool matrix = false) {
    std::vector<SignatureParam> ps{image_in("in")};
    if (matrix) ps.push_back(param(Direction::Input, ObjKind::Matrix, "mask"));
    ps.push_back(image_out("out", {out_fmt}));
    std::vector<ObjectId> args = ins;
    args.push_back(out);
    a.impl->add_abstraction_node(make_local_kernel(label, KernelSignature(std::move(ps)), std::move(lk)),
                                 args, a.node->id, label);
}

std::vector<Value> ints(std::initializer_list<std::int64_t> v) {
    std::vector<Value> out;
    for (std::int64_t x : v) out.push_back(Value::of_int(x));
    return out;
}

/// 3x3 Sum window of mask(0,0) * win(0,0,0) under Clamp, with a post body.
LocalKernel masked3x3(std::vector<Value> mask, bool real, ExprPtr post) {
    LocalKernel lk;
    lk.window_w = lk.window_h = 3;
    lk.boundary = BoundaryMode::Clamp;
    lk.combine = CombineMode::Sum;
    lk.tap_body = mul(mask_coef(0, 0), window_pixel(0, 0, 0));
    lk.mask = std::move(mask);
    lk.mask_is_real = real;
    lk.post_body = std::move(post);
    return lk;
}

// Float Gaussian mask used when the image is F32 (Listing 2 of the paper).
const double kGaussianF32[9] = {0.057118, 0.124758, 0.057118, 0.124758, 0.272496,
                                0.124758, 0.057118, 0.124758, 0.057118};

KernelEntry entry(std::string name, std::vector<SignatureParam> params,
                  std::function<std::vector<ResolvedDesc>(const InferArgs&)> infer,
                  std::function<void(ExpandArgs&)> expand) {
    KernelEntry e;
    e.name = std::move(name);
    e.signature = KernelSignature(std::move(params));
    e.infer = std::move(infer);
    e.expand = std::move(expand);
    return e;
}

// ======================================================================= points

void add_points(KernelRegistry& r) {
    r.add(entry(
        "ChannelExtract",
        {image_in("in", {ImageFormat::UYVY, ImageFormat::RGB}), image_out("out", {ImageFormat::U8})},
        [](const InferArgs& a) {
            const Channel c = get_channel(*a.attrs);
            const ImageFormat f = a.inputs[0].format;
            if (f == ImageFormat::UYVY && c != Channel::Y)
                throw Error(ErrorCode::BadFormat, "UYVY extraction supports channel Y only");
            if (f == ImageFormat::RGB && !(c == Channel::R || c == Channel::G || c == Channel::B))
                throw Error(ErrorCode::BadFormat, "RGB extraction needs channel R, G or B");
            return like_input(a, ImageFormat::U8);
        },
        [](ExpandArgs& a) {
            const Channel c = get_channel(a.node->attrs);
            point_node(a, std::string("extract_") + to_string(c), ImageFormat::U8, input_pixel(0, c),
                       {a.input_ids[0]}, a.output_ids[0]);
        }));

    r.add(entry(
        "ChannelCombine",
        {image_in("r", {ImageFormat::U8}), image_in("g", {ImageFormat::U8}),
         image_in("b", {ImageFormat::U8}), image_out("out", {ImageFormat::RGB})},
        [](const InferArgs& a) {
            same_dims(a.inputs);
            return like_input(a, ImageFormat::RGB);
        },
        [](ExpandArgs& a) {
            PointKernel pk;
            pk.arity = 3;
            pk.outputs.push_back(PointOutput{{px(0), px(1), px(2)}});
            std::vector<SignatureParam> ps{param(Direction::Input, ObjKind::Image, "in0"),
                                           param(Direction::Input, ObjKind::Image, "in1"),
                                           param(Direction::Input, ObjKind::Image, "in2"),
                                           image_out("out", {ImageFormat::RGB})};
            a.impl->add_abstraction_node(
                make_point_kernel("combine_rgb", KernelSignature(std::move(ps)), std::move(pk)),
                {a.input_ids[0], a.input_ids[1], a.input_ids[2], a.output_ids[0]}, a.node->id,
                "combine_rgb");
        }));

    struct Arith {
        const char* name;
        const char* label;
        ExprOp op;
    };
    for (Arith ar : {Arith{"Add", "add", ExprOp::Add}, Arith{"Subtract", "subtract", ExprOp::Sub},
                     Arith{"Multiply", "multiply", ExprOp::Mul}}) {
        const bool prod = ar.op == ExprOp::Mul;
        auto default_fmt = [prod](const std::vector<ResolvedDesc>& in) {
            return prod ? product_result(in[0].format, in[1].format)
                        : sum_result(in[0].format, in[1].format);
        };
        r.add(entry(
            ar.name, {image_in("in0", single_channel()), image_in("in1", single_channel()), image_out("out")},
            [default_fmt](const InferArgs& a) {
                same_dims(a.inputs);
                return like_input(a, get_format(*a.attrs, "out", default_fmt(a.inputs)));
            },
            [ar, prod, default_fmt](ExpandArgs& a) {
                const ImageFormat out = get_format(a.node->attrs, "out", default_fmt(a.inputs));
                ExprPtr body = binary(ar.op, px(0), px(1));
                if (prod) {
                    const double s = get_real(a.node->attrs, "scale", 1.0);
                    if (s != 1.0) body = mul(std::move(body), const_f(s));
                }
                point_node(a, ar.label, out, saturate_to(scalar_of(out), std::move(body)),
                           {a.input_ids[0], a.input_ids[1]}, a.output_ids[0]);
            }));
    }

    r.add(entry(
        "AbsDiff", {image_in("in0", integer_channel()), image_in("in1", integer_channel()), image_out("out")},
        [](const InferArgs& a) {
            same_dims(a.inputs);
            if (a.inputs[0].format != a.inputs[1].format)
                throw Error(ErrorCode::BadFormat, "AbsDiff needs matching input formats");
            return like_input(a, a.inputs[0].format);
        },
        [](ExpandArgs& a) {
            const ImageFormat f = a.inputs[0].format;
            point_node(a, "absdiff", f, saturate_to(scalar_of(f), unary(ExprOp::Abs, sub(px(0), px(1)))),
                       {a.input_ids[0], a.input_ids[1]}, a.output_ids[0]);
        }));

    struct Bit {
        const char* name;
        const char* label;
        ExprOp op;
    };
    for (Bit bt : {Bit{"And", "and", ExprOp::And}, Bit{"Or", "or", ExprOp::Or},
                   Bit{"Xor", "xor", ExprOp::Xor}}) {
        const std::string nm = bt.name;
        r.add(entry(
            bt.name, {image_in("in0", integer_channel()), image_in("in1", integer_channel()), image_out("out")},
            [nm](const InferArgs& a) {
                same_dims(a.inputs);
                if (a.inputs[0].format != a.inputs[1].format)
                    throw Error(ErrorCode::BadFormat, nm + " needs matching input formats");
                return like_input(a, a.inputs[0].format);
            },
            [bt](ExpandArgs& a) {
                const ImageFormat f = a.inputs[0].format;
                point_node(a, bt.label, f, cast(scalar_of(f), CastPolicy::Wrap, binary(bt.op, px(0), px(1))),
                           {a.input_ids[0], a.input_ids[1]}, a.output_ids[0]);
            }));
    }

    r.add(entry(
        "Not", {image_in("in", integer_channel()), image_out("out")},
        [](const InferArgs& a) { return like_input(a, a.inputs[0].format); },
        [](ExpandArgs& a) {
            const ImageFormat f = a.inputs[0].format;
            point_node(a, "not", f, cast(scalar_of(f), CastPolicy::Wrap, unary(ExprOp::Not, px(0))),
                       {a.input_ids[0]}, a.output_ids[0]);
        }));

    r.add(entry(
        "Magnitude",
        {image_in("gx", {ImageFormat::S16}), image_in("gy", {ImageFormat::S16}),
         image_out("out", {ImageFormat::S16})},
        [](const InferArgs& a) {
            same_dims(a.inputs);
            return like_input(a, ImageFormat::S16);
        },
        [](ExpandArgs& a) {
            ExprPtr body = saturate_to(ScalarType::S16,
                                       unary(ExprOp::Sqrt, add(mul(px(0), px(0)), mul(px(1), px(1)))));
            point_node(a, "magnitude", ImageFormat::S16, std::move(body), {a.input_ids[0], a.input_ids[1]},
                       a.output_ids[0]);
        }));

    r.add(entry(
        "Phase",
        {image_in("gx", {ImageFormat::S16}), image_in("gy", {ImageFormat::S16}),
         image_out("out", {ImageFormat::U8})},
        [](const InferArgs& a) {
            same_dims(a.inputs);
            return like_input(a, ImageFormat::U8);
        },
        [](ExpandArgs& a) {
            ExprPtr ang = binary(ExprOp::Atan2, px(1), px(0));
            ExprPtr pos = select(binary(ExprOp::Lt, ang, const_f(0.0)), add(ang, const_f(kTau)), ang);
            ExprPtr q = add(mul(std::move(pos), const_f(256.0 / kTau)), const_f(0.5));
            point_node(a, "phase", ImageFormat::U8, cast(ScalarType::U8, CastPolicy::Wrap, std::move(q)),
                       {a.input_ids[0], a.input_ids[1]}, a.output_ids[0]);
        }));

    {
        SignatureParam upper = param(Direction::Input, ObjKind::Scalar, "upper");
        upper.state = ParamState::Optional;
        r.add(entry(
            "Threshold",
            {image_in("in", integer_channel()), param(Direction::Input, ObjKind::Scalar, "thresh"), upper,
             image_out("out", {ImageFormat::U8})},
            [](const InferArgs& a) {
                const std::string mode = get_str(*a.attrs, "mode", "binary");
                if (mode != "binary" && mode != "range")
                    throw Error(ErrorCode::SchemaError, "threshold mode must be binary or range");
                scalar_within(*a.ctx, *a.node, 1, a.inputs[0].format);
                scalar_within(*a.ctx, *a.node, 2, a.inputs[0].format);
                return like_input(a, ImageFormat::U8);
            },
            [](ExpandArgs& a) {
                const std::string mode = get_str(a.node->attrs, "mode", "binary");
                if (mode == "binary" || a.input_ids[2] == kInvalidId) {
                    ExprPtr body = saturate_to(ScalarType::U8, select(binary(ExprOp::Gt, px(0), px(1)),
                                                                      const_i(255), const_i(0)));
                    point_node(a, "threshold", ImageFormat::U8, std::move(body),
                               {a.input_ids[0], a.input_ids[1]}, a.output_ids[0],
                               {ObjKind::Image, ObjKind::Scalar});
                    return;
                }
                ExprPtr outside = binary(ExprOp::Or, binary(ExprOp::Lt, px(0), px(1)),
                                         binary(ExprOp::Gt, px(0), px(2)));
                ExprPtr body = saturate_to(ScalarType::U8, select(std::move(outside), const_i(0), const_i(255)));
                point_node(a, "threshold_range", ImageFormat::U8, std::move(body),
                           {a.input_ids[0], a.input_ids[1], a.input_ids[2]}, a.output_ids[0],
                           {ObjKind::Image, ObjKind::Scalar, ObjKind::Scalar});
            }));
    }

    r.add(entry(
        "ConvertDepth", {image_in("in", integer_channel()), image_out("out")},
        [](const InferArgs& a) {
            const ImageFormat to = get_format(*a.attrs, "to", ImageFormat::U8);
            if (to == ImageFormat::F32 || to == ImageFormat::RGB || to == ImageFormat::UYVY)
                throw Error(ErrorCode::BadFormat, "depth conversion targets integer formats");
            return like_input(a, to);
        },
        [](ExpandArgs& a) {
            const ImageFormat to = get_format(a.node->attrs, "to", ImageFormat::U8);
            const std::int64_t shift = get_int(a.node->attrs, "shift", 0);
            const CastPolicy pol = get_str(a.node->attrs, "policy", "saturate") == "wrap"
                                       ? CastPolicy::Wrap
                                       : CastPolicy::Saturate;
            ExprPtr body = px(0);
            if (shift > 0) {
                const bool widening = bytes_per_pixel(to) >= bytes_per_pixel(a.inputs[0].format);
                body = binary(widening ? ExprOp::Shl : ExprOp::Shr, std::move(body), const_i(shift));
            }
            point_node(a, "convert_depth", to, cast(scalar_of(to), pol, std::move(body)), {a.input_ids[0]},
                       a.output_ids[0]);
        }));

    r.add(entry(
        "Copy", {image_in("in"), image_out("out")},
        [](const InferArgs& a) {
            if (a.inputs[0].format == ImageFormat::UYVY)
                throw Error(ErrorCode::BadFormat, "Copy does not support packed UYVY");
            return like_input(a, a.inputs[0].format);
        },
        [](ExpandArgs& a) {
            if (a.inputs[0].format != ImageFormat::RGB) {
                point_node(a, "copy", a.inputs[0].format, px(0), {a.input_ids[0]}, a.output_ids[0]);
                return;
            }
            PointKernel pk;
            pk.arity = 1;
            pk.outputs.push_back(PointOutput{{input_pixel(0, Channel::R), input_pixel(0, Channel::G),
                                              input_pixel(0, Channel::B)}});
            std::vector<SignatureParam> ps{param(Direction::Input, ObjKind::Image, "in0"),
                                           image_out("out", {ImageFormat::RGB})};
            a.impl->add_abstraction_node(make_point_kernel("copy", KernelSignature(std::move(ps)), std::move(pk)),
                                         {a.input_ids[0], a.output_ids[0]}, a.node->id, "copy");
        }));
}

// ======================================================================= locals

void add_locals(KernelRegistry& r) {
    r.add(entry(
        "Box3x3", {image_in("in", single_channel()), image_out("out")},
        [](const InferArgs& a) { return like_input(a, a.inputs[0].format); },
        [](ExpandArgs& a) {
            const ImageFormat f = a.inputs[0].format;
            local_node(a, "box3x3", f,
                       masked3x3(ints({1, 1, 1, 1, 1, 1, 1, 1, 1}), false,
                                 saturate_to(scalar_of(f), mul(px(0), const_f(1.0 / 9.0)))),
                       {a.input_ids[0]}, a.output_ids[0]);
        }));

    r.add(entry(
        "Gaussian3x3", {image_in("in", single_channel()), image_out("out")},
        [](const InferArgs& a) { return like_input(a, a.inputs[0].format); },
        [](ExpandArgs& a) {
            const ImageFormat f = a.inputs[0].format;
            LocalKernel lk;
            if (f == ImageFormat::F32) {
                std::vector<Value> m;
                for (double c : kGaussianF32) m.push_back(Value::of_real(c));
                lk = masked3x3(std::move(m), true, saturate_to(scalar_of(f), px(0)));
            } else {
                lk = masked3x3(ints({1, 2, 1, 2, 4, 2, 1, 2, 1}), false,
                               saturate_to(scalar_of(f), mul(px(0), const_f(1.0 / 16.0))));
            }
            local_node(a, "gaussian3x3", f, std::move(lk), {a.input_ids[0]}, a.output_ids[0]);
        }));

    r.add(entry(
        "Sobel3x3",
        {image_in("in", {ImageFormat::U8}), image_out("gx", {ImageFormat::S16}, ParamState::Optional),
         image_out("gy", {ImageFormat::S16}, ParamState::Optional)},
        [](const InferArgs& a) {
            ResolvedDesc d = img_desc(a.inputs[0].width, a.inputs[0].height, ImageFormat::S16);
            return std::vector<ResolvedDesc>{d, d};
        },
        [](ExpandArgs& a) {
            auto sobel = [](std::initializer_list<std::int64_t> m) {
                return masked3x3(ints(m), false, saturate_to(ScalarType::S16, px(0)));
            };
            if (a.output_ids[0] != kInvalidId)
                local_node(a, "sobel_x", ImageFormat::S16, sobel({-1, 0, 1, -2, 0, 2, -1, 0, 1}),
                           {a.input_ids[0]}, a.output_ids[0]);
            if (a.output_ids[1] != kInvalidId)
                local_node(a, "sobel_y", ImageFormat::S16, sobel({-1, -2, -1, 0, 0, 0, 1, 2, 1}),
                           {a.input_ids[0]}, a.output_ids[1]);
        }));

    auto window_op = [&r](const char* name, const char* label, CombineMode comb, bool median) {
        r.add(entry(
            name, {image_in("in", integer_channel()), image_out("out")},
            [](const InferArgs& a) { return like_input(a, a.inputs[0].format); },
            [label, comb, median](ExpandArgs& a) {
                const ImageFormat f = a.inputs[0].format;
                LocalKernel lk;
                lk.window_w = lk.window_h = 3;
                lk.boundary = BoundaryMode::Clamp;
                lk.combine = comb;
                lk.median3x3 = median;
                lk.tap_body = window_pixel(0, 0, 0);
                lk.post_body = saturate_to(scalar_of(f), px(0));
                local_node(a, label, f, std::move(lk), {a.input_ids[0]}, a.output_ids[0]);
            }));
    };
    window_op("Dilate3x3", "dilate3x3", CombineMode::Max, false);
    window_op("Erode3x3", "erode3x3", CombineMode::Min, false);
    window_op("Median3x3", "median3x3", CombineMode::Min, true);

    auto conv_default = [](const std::vector<ResolvedDesc>& in) {
        if (is_float(in[1].element_type) || in[0].format == ImageFormat::F32) return ImageFormat::F32;
        return in[0].format == ImageFormat::S32 ? ImageFormat::S32 : ImageFormat::S16;
    };
    r.add(entry(
        "Convolve",
        {image_in("in", single_channel()), param(Direction::Input, ObjKind::Matrix, "matrix"), image_out("out")},
        [conv_default](const InferArgs& a) {
            const ResolvedDesc& m = a.inputs[1];
            if (m.rows % 2 == 0 || m.cols % 2 == 0)
                throw Error(ErrorCode::BadFormat, "convolution matrix must have odd dimensions");
            return like_input(a, get_format(*a.attrs, "out", conv_default(a.inputs)));
        },
        [conv_default](ExpandArgs& a) {
            const ResolvedDesc& m = a.inputs[1];
            const ImageFormat out = get_format(a.node->attrs, "out", conv_default(a.inputs));
            const std::int64_t scale = get_int(a.node->attrs, "scale", 1);
            if (scale < 1) throw Error(ErrorCode::SchemaError, "convolve scale must be >= 1");
            LocalKernel lk;
            lk.window_w = m.cols;
            lk.window_h = m.rows;
            lk.boundary = BoundaryMode::Clamp;
            lk.combine = CombineMode::Sum;
            lk.tap_body = mul(mask_coef(0, 0), window_pixel(0, 0, 0));
            ExprPtr v = px(0);
            if (scale != 1) v = mul(std::move(v), const_f(1.0 / static_cast<double>(scale)));
            lk.post_body = saturate_to(scalar_of(out), std::move(v));
            local_node(a, "convolve", out, std::move(lk), {a.input_ids[0], a.input_ids[1]}, a.output_ids[0],
                       true);
        }));
}

// ====================================================================== globals

AbstractionPtr histogram_kernel(std::int64_t bins, std::int64_t offset, std::int64_t range) {
    AbstractionKernel t;
    HistogramKernel hk;
    hk.bins = static_cast<int>(bins);
    hk.offset = offset;
    hk.range = range;
    hk.bin_of = div(mul(sub(px(0), const_i(offset)), const_i(bins)), const_i(range));
    t.body = hk;
    return make_kernel("histogram", AbstractionKind::Histogram,
                       KernelSignature({image_in("in", {ImageFormat::U8}),
                                        param(Direction::Output, ObjKind::Array, "dist", {}, ScalarType::S32)}),
                       t);
}

void add_globals(KernelRegistry& r) {
    r.add(entry(
        "Histogram",
        {image_in("in", {ImageFormat::U8}), param(Direction::Output, ObjKind::Array, "dist", {}, ScalarType::S32)},
        [](const InferArgs& a) {
            const std::int64_t bins = get_int(*a.attrs, "bins", 256);
            if (bins < 1) throw Error(ErrorCode::SchemaError, "histogram needs bins >= 1");
            return std::vector<ResolvedDesc>{array_desc(ScalarType::S32, bins)};
        },
        [](ExpandArgs& a) {
            AbstractionPtr k = histogram_kernel(get_int(a.node->attrs, "bins", 256),
                                                get_int(a.node->attrs, "offset", 0),
                                                get_int(a.node->attrs, "range", 256));
            a.impl->add_abstraction_node(k, {a.input_ids[0], a.output_ids[0]}, a.node->id, "histogram");
        }));

    r.add(entry(
        "MinMaxLoc",
        {image_in("in", integer_channel()),
         param(Direction::Output, ObjKind::Scalar, "min", {}, ScalarType::U8),
         param(Direction::Output, ObjKind::Scalar, "max", {}, ScalarType::U8),
         param(Direction::Output, ObjKind::Array, "minloc", {}, ScalarType::S32, ParamState::Optional),
         param(Direction::Output, ObjKind::Array, "maxloc", {}, ScalarType::S32, ParamState::Optional)},
        [](const InferArgs& a) {
            const ScalarType t = scalar_of(a.inputs[0].format);
            return std::vector<ResolvedDesc>{scalar_desc(t), scalar_desc(t), array_desc(ScalarType::S32, 2),
                                             array_desc(ScalarType::S32, 2)};
        },
        [](ExpandArgs& a) {
            const ScalarType t = scalar_of(a.inputs[0].format);
            for (bool lo : {true, false}) {
                AbstractionKernel tpl;
                ReduceKernel rk;
                rk.seed_first = true;
                rk.combine = binary(lo ? ExprOp::Min : ExprOp::Max, px(0), px(1));
                rk.finalize = saturate_to(t, px(0));
                rk.track = lo ? ReduceKernel::Track::ArgMin : ReduceKernel::Track::ArgMax;
                tpl.body = rk;
                const char* nm = lo ? "reduce_min" : "reduce_max";
                AbstractionPtr k = make_kernel(
                    nm, AbstractionKind::Reduce,
                    KernelSignature({image_in("in"), param(Direction::Output, ObjKind::Scalar, "value", {}, t),
                                     param(Direction::Output, ObjKind::Array, "loc", {}, ScalarType::S32,
                                           ParamState::Optional)}),
                    tpl);
                a.impl->add_abstraction_node(
                    k, {a.input_ids[0], a.output_ids[lo ? 0 : 1], a.output_ids[lo ? 2 : 3]}, a.node->id, nm);
            }
        }));

    r.add(entry(
        "MeanStdDev",
        {image_in("in", integer_channel()),
         param(Direction::Output, ObjKind::Scalar, "mean", {}, ScalarType::F32),
         param(Direction::Output, ObjKind::Scalar, "stddev", {}, ScalarType::F32)},
        [](const InferArgs&) {
            return std::vector<ResolvedDesc>{scalar_desc(ScalarType::F32), scalar_desc(ScalarType::F32)};
        },
        [](ExpandArgs& a) {
            // mean = float(sum * 1.0 / n)
            AbstractionKernel mt;
            {
                ReduceKernel rk;
                rk.init = Value::of_int(0);
                rk.combine = add(px(0), px(1));
                rk.finalize = saturate_to(ScalarType::F32, div(mul(px(0), const_f(1.0)), px(1)));
                mt.body = rk;
            }
            a.impl->add_abstraction_node(
                make_kernel("reduce_mean", AbstractionKind::Reduce,
                            KernelSignature({image_in("in"),
                                             param(Direction::Output, ObjKind::Scalar, "mean", {}, ScalarType::F32)}),
                            mt),
                {a.input_ids[0], a.output_ids[0]}, a.node->id, "reduce_mean");
            // stddev = float(sqrt(max(sumsq * 1.0 / n - mean_f * mean_f, 0)))
            AbstractionKernel st;
            {
                ReduceKernel rk;
                rk.init = Value::of_int(0);
                rk.combine = add(px(0), mul(px(1), px(1)));
                ExprPtr var = binary(ExprOp::Max, sub(div(mul(px(0), const_f(1.0)), px(1)), mul(px(2), px(2))),
                                     const_f(0.0));
                rk.finalize = saturate_to(ScalarType::F32, unary(ExprOp::Sqrt, std::move(var)));
                rk.extra_scalar_inputs = 1;
                st.body = rk;
            }
            a.impl->add_abstraction_node(
                make_kernel("reduce_stddev", AbstractionKind::Reduce,
                            KernelSignature({image_in("in"), param(Direction::Input, ObjKind::Scalar, "mean"),
                                             param(Direction::Output, ObjKind::Scalar, "stddev", {},
                                                   ScalarType::F32)}),
                            st),
                {a.input_ids[0], a.output_ids[0], a.output_ids[1]}, a.node->id, "reduce_stddev");
        }));

    r.add(entry(
        "IntegralImage", {image_in("in", {ImageFormat::U8}), image_out("out", {ImageFormat::S32})},
        [](const InferArgs& a) { return like_input(a, ImageFormat::S32); },
        [](ExpandArgs& a) {
            AbstractionKernel t;
            t.body = ScanKernel{};
            a.impl->add_abstraction_node(
                make_kernel("integral", AbstractionKind::Scan,
                            KernelSignature({image_in("in", {ImageFormat::U8}), image_out("out", {ImageFormat::S32})}),
                            t),
                {a.input_ids[0], a.output_ids[0]}, a.node->id, "integral");
        }));

    r.add(entry(
        "ScaleImage", {image_in("in", {ImageFormat::U8, ImageFormat::S16, ImageFormat::F32}), image_out("out")},
        [](const InferArgs& a) {
            const Binding* b = a.node->binding_for(1);
            const DataObject* o = b ? a.ctx->find(b->object) : nullptr;
            if (!o || o->width < 1 || o->height < 1)
                throw Error(ErrorCode::BadFormat, "scale output needs explicit dimensions");
            return std::vector<ResolvedDesc>{img_desc(o->width, o->height, a.inputs[0].format)};
        },
        [](ExpandArgs& a) {
            const std::string interp = get_str(a.node->attrs, "interp", "nearest");
            AbstractionKernel t;
            ScaleKernel sk;
            sk.interp = interp == "bilinear" ? InterpMode::Bilinear : InterpMode::Nearest;
            t.body = sk;
            const std::string nm = "scale_" + interp;
            a.impl->add_abstraction_node(
                make_kernel(nm, AbstractionKind::Scale,
                            KernelSignature({image_in("in"), image_out("out", {a.inputs[0].format})}), t),
                {a.input_ids[0], a.output_ids[0]}, a.node->id, nm);
        }));

    r.add(entry(
        "EqualizeHist", {image_in("in", {ImageFormat::U8}), image_out("out", {ImageFormat::U8})},
        [](const InferArgs& a) { return like_input(a, ImageFormat::U8); },
        [](ExpandArgs& a) {
            Context& ctx = *a.ctx;
            DataObject& hist = ctx.create_virtual_object(*a.impl, ObjKind::Array, "eq_hist");
            hist.element_type = ScalarType::S32;
            hist.capacity = 256;
            DataObject& lut = ctx.create_virtual_object(*a.impl, ObjKind::Array, "eq_lut");
            lut.element_type = ScalarType::U8;
            lut.capacity = 256;
            a.impl->add_abstraction_node(histogram_kernel(256, 0, 256), {a.input_ids[0], hist.id}, a.node->id,
                                         "histogram");
            AbstractionKernel t;
            t.body = TableKernel{TableKernel::Fn::EqualizeHistLut};
            a.impl->add_abstraction_node(
                make_kernel("equalize_lut", AbstractionKind::Table,
                            KernelSignature({param(Direction::Input, ObjKind::Array, "dist", {}, ScalarType::S32),
                                             param(Direction::Output, ObjKind::Array, "lut", {}, ScalarType::U8)}),
                            t),
                {hist.id, lut.id}, a.node->id, "equalize_lut");
            point_node(a, "lut_lookup", ImageFormat::U8, array_at(1, px(0)), {a.input_ids[0], lut.id},
                       a.output_ids[0], {ObjKind::Image, ObjKind::Array});
        }));
}

} // namespace

ExprPtr saturate_to(ScalarType t, ExprPtr e) { return cast(t, CastPolicy::Saturate, std::move(e)); }

// ------------------------------------------------------------- abstraction infer

std::vector<ResolvedDesc> infer_abstraction(const AbstractionKernel& k, const InferArgs& args,
                                            std::vector<ScalarType>* types_out) {
    const std::vector<ScalarType> types = typecheck(k, args.inputs);
    if (types_out) *types_out = types;
    if (k.kind == AbstractionKind::Point || k.kind == AbstractionKind::Local) same_dims(args.inputs);

    ResolvedDesc src;
    for (const ResolvedDesc& d : args.inputs)
        if (d.kind == ObjKind::Image) {
            src = d;
            break;
        }

    std::vector<ResolvedDesc> outs;
    std::size_t oi = 0;
    for (std::size_t pi = 0; pi < k.signature.params.size(); ++pi) {
        const SignatureParam& p = k.signature.params[pi];
        if (p.direction != Direction::Output) continue;
        ResolvedDesc d;
        d.kind = p.kind;
        const ScalarType t = oi < types.size() ? types[oi] : p.element_type;
        switch (k.kind) {
        case AbstractionKind::Point:
        case AbstractionKind::Local:
        case AbstractionKind::Scan:
            d.width = src.width;
            d.height = src.height;
            d.format = p.formats.size() == 1 ? p.formats.front() : format_of(t);
            break;
        case AbstractionKind::Scale: {
            const Binding* b = args.node ? args.node->binding_for(static_cast<int>(pi)) : nullptr;
            const DataObject* o = (b && args.ctx) ? args.ctx->find(b->object) : nullptr;
            if (!o || o->width < 1 || o->height < 1)
                throw Error(ErrorCode::BadFormat, "scale output needs explicit dimensions");
            d.width = o->width;
            d.height = o->height;
            d.format = src.format;
            break;
        }
        case AbstractionKind::Reduce:
            d.element_type = t;
            d.capacity = p.kind == ObjKind::Array ? 2 : 0;
            break;
        case AbstractionKind::Histogram:
            d.element_type = ScalarType::S32;
            d.capacity = k.histogram().bins;
            break;
        case AbstractionKind::Table:
            d.element_type = p.element_type;
            d.capacity = 256;
            break;
        }
        if (d.kind == ObjKind::Scalar) d.element_type = t;
        outs.push_back(d);
        ++oi;
    }
    return outs;
}

// ------------------------------------------------------------------ registry

const KernelEntry* KernelRegistry::find(const std::string& name) const {
    auto it = entries_.find(name);
    return it == entries_.end() ? nullptr : &it->second;
}

std::vector<std::string> KernelRegistry::names() const {
    std::vector<std::string> out;
    out.reserve(entries_.size());
    for (const auto& kv : entries_) out.push_back(kv.first);
    return out;
}

void KernelRegistry::add(KernelEntry e) {
    std::string key = e.name;
    entries_[key] = std::move(e);
}

void KernelRegistry::add_custom(AbstractionPtr kernel) {
    KernelEntry e;
    e.name = kernel->name;
    e.signature = kernel->signature;
    e.infer = [kernel](const InferArgs& a) { return infer_abstraction(*kernel, a); };
    e.expand = [kernel](ExpandArgs& a) {
        std::vector<ObjectId> args;
        std::size_t ii = 0, oi = 0;
        for (const SignatureParam& p : kernel->signature.params)
            args.push_back(p.direction == Direction::Input ? a.input_ids[ii++] : a.output_ids[oi++]);
        a.impl->add_abstraction_node(kernel, args, a.node->id, kernel->name);
    };
    add(std::move(e));
}

const KernelRegistry& KernelRegistry::builtin() {
    static const KernelRegistry reg = [] {
        KernelRegistry r;
        add_points(r);
        add_locals(r);
        add_globals(r);
        return r;
    }();
    return reg;
}

// -------------------------------------------------------------------- expand

AppGraph& expand(const VerifiedGraph& vg, Context& ctx) {
    if (!vg.stamped()) throw Error(ErrorCode::UnstampedGraph, "expand needs a verified graph");
    const AppGraph& src = vg.graph();
    AppGraph& impl = ctx.create_graph(GraphPhase::Implementation);
    impl.derive_from(src);

    if (src.phase() == GraphPhase::Implementation) {
        for (ObjectId d : src.data()) impl.note_data(d);
        for (ObjectId nid : src.topo_sort()) {
            OperatorNode copy = *src.node(nid);
            copy.id = kInvalidId;
            impl.add_node_unchecked(std::move(copy));
        }
        return impl;
    }

    const KernelRegistry& reg = ctx.registry();
    for (ObjectId nid : src.topo_sort()) {
        const OperatorNode* n = src.node(nid);
        const KernelEntry* e = reg.find(n->kernel);
        if (!e) throw Error(ErrorCode::UnknownKernel, "kernel '" + n->kernel + "' is not registered", n->id);
        ExpandArgs a;
        a.impl = &impl;
        a.ctx = &ctx;
        a.node = n;
        for (std::size_t i = 0; i < e->signature.params.size(); ++i) {
            const Binding* b = n->binding_for(static_cast<int>(i));
            const ObjectId id = b ? b->object : kInvalidId;
            if (e->signature.params[i].direction == Direction::Input) {
                a.input_ids.push_back(id);
                a.inputs.push_back(id == kInvalidId ? ResolvedDesc{} : vg.desc(id));
            } else {
                a.output_ids.push_back(id);
            }
        }
        e->expand(a);
    }
    return impl;
}

} // namespace gvx
