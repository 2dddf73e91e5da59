// The five BASELINE.json configurations as OpenVX-style graphs, written only
// against the public graph API so the same source builds against graphvx-b200
// (namespace gvx) and against the unmodified reference compiled with
// -Dgvx=gvxref (oracle/ref_shim.cpp).  Definitions fixed by SURVEY.md §8a /
// §8d:
//   cfg1 / cfg5  Gaussian3x3 -> Sobel3x3 -> Magnitude (U8 -> S16)
//   cfg2         Harris: Sobel3x3 -> Multiply gx*gx, gy*gy, gx*gy (S32) ->
//                Box3x3 x3 -> user point HarrisResponse (F32) -> user point
//                ThresholdF32 (U8 mask)
//   cfg3         unsharp mask: user-defined 5x5 local Blur5x5 (binomial /256)
//                -> Subtract(in, blur) -> Add(in, diff) -> ConvertDepth (U8)
//   cfg4         Convolve(5x5 binomial, scale 256) -> ConvertDepth (U8) ->
//                Histogram(256) + MeanStdDev
// `virtual_mid` selects virtual intermediates (graphvx-b200) or plain images
// (needed by the reference, whose expand() rejects virtual images,
// SURVEY.md §0 finding 1; run_naive semantics are identical).
#pragma once

#include "graphvx/execute.hpp"
#include "graphvx/registry.hpp"
#include "graphvx/verify.hpp"

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace gvx_configs {

struct ConfigGraph {
    gvx::AppGraph* graph = nullptr;
    gvx::ObjectId input = gvx::kInvalidId;
    std::vector<gvx::ObjectId> outputs; // final results, in config order
};

constexpr double kHarrisK = 0.04;
constexpr double kHarrisThreshold = 1.0e9;

inline gvx::AbstractionPtr harris_response_kernel() {
    using namespace gvx;
    std::vector<SignatureParam> ps(4);
    const char* names[] = {"sxx", "syy", "sxy", "resp"};
    for (int i = 0; i < 4; ++i) {
        ps[static_cast<std::size_t>(i)].direction = i < 3 ? Direction::Input : Direction::Output;
        ps[static_cast<std::size_t>(i)].kind = ObjKind::Image;
        ps[static_cast<std::size_t>(i)].name = names[i];
    }
    ps[0].formats = ps[1].formats = ps[2].formats = {ImageFormat::S32};
    ps[3].formats = {ImageFormat::F32};
    const ExprPtr a = input_pixel(0), b = input_pixel(1), c = input_pixel(2);
    const ExprPtr det = sub(mul(a, b), mul(c, c));
    const ExprPtr tr = add(a, b);
    PointKernel pk;
    pk.arity = 3;
    pk.outputs.push_back(PointOutput{{cast(ScalarType::F32, CastPolicy::Saturate,
                                           sub(det, mul(const_f(kHarrisK), mul(tr, tr))))}});
    return make_point_kernel("HarrisResponse", KernelSignature(ps), pk);
}

inline gvx::AbstractionPtr threshold_f32_kernel(double t) {
    using namespace gvx;
    std::vector<SignatureParam> ps(2);
    ps[0].direction = Direction::Input;
    ps[0].kind = ObjKind::Image;
    ps[0].formats = {ImageFormat::F32};
    ps[0].name = "resp";
    ps[1].direction = Direction::Output;
    ps[1].kind = ObjKind::Image;
    ps[1].formats = {ImageFormat::U8};
    ps[1].name = "mask";
    PointKernel pk;
    pk.arity = 1;
    pk.outputs.push_back(PointOutput{{cast(ScalarType::U8, CastPolicy::Saturate,
                                           select(binary(ExprOp::Gt, input_pixel(0), const_f(t)), const_i(255),
                                                  const_i(0)))}});
    return make_point_kernel("ThresholdF32", KernelSignature(ps), pk);
}

inline const std::vector<std::int64_t>& binomial5() {
    static const std::vector<std::int64_t> m = {1, 4,  6,  4,  1, 4, 16, 24, 16, 4, 6, 24, 36,
                                                24, 6, 4, 16, 24, 16, 4,  1, 4,  6, 4, 1};
    return m;
}

inline gvx::AbstractionPtr blur5x5_kernel() {
    using namespace gvx;
    std::vector<SignatureParam> ps(2);
    ps[0].direction = Direction::Input;
    ps[0].kind = ObjKind::Image;
    ps[0].formats = {ImageFormat::U8};
    ps[0].name = "in";
    ps[1].direction = Direction::Output;
    ps[1].kind = ObjKind::Image;
    ps[1].formats = {ImageFormat::U8};
    ps[1].name = "out";
    LocalKernel lk;
    lk.window_w = lk.window_h = 5;
    lk.boundary = BoundaryMode::Clamp;
    lk.combine = CombineMode::Sum;
    lk.tap_body = mul(mask_coef(0, 0), window_pixel(0, 0, 0));
    for (std::int64_t v : binomial5()) lk.mask.push_back(Value::of_int(v));
    lk.post_body = cast(ScalarType::U8, CastPolicy::Saturate, mul(input_pixel(0), const_f(1.0 / 256.0)));
    return make_local_kernel("Blur5x5", KernelSignature(ps), lk);
}

/// Registers the user-defined kernels of cfg2 / cfg3 on the context.
inline void install_custom_kernels(gvx::Context& ctx) {
    auto reg = std::make_shared<gvx::KernelRegistry>(gvx::KernelRegistry::builtin().clone());
    reg->add_custom(harris_response_kernel());
    reg->add_custom(threshold_f32_kernel(kHarrisThreshold));
    reg->add_custom(blur5x5_kernel());
    ctx.set_registry(reg);
}

inline ConfigGraph build_config(gvx::Context& ctx, int cfg, int w, int h, bool virtual_mid) {
    using namespace gvx;
    install_custom_kernels(ctx);
    ConfigGraph cg;
    AppGraph& g = ctx.create_graph();
    cg.graph = &g;
    auto image = [&](ImageFormat f, const char* name) {
        ObjectId id = ctx.create_image(w, h, f, name).id;
        g.note_data(id);
        return id;
    };
    auto mid = [&](ImageFormat f, const char* name) {
        return virtual_mid ? ctx.create_virtual_image(g, name).id : image(f, name);
    };
    cg.input = image(ImageFormat::U8, "in");
    switch (cfg) {
    case 1:
    case 5: {
        ObjectId gs = mid(ImageFormat::U8, "gauss");
        ObjectId gx = mid(ImageFormat::S16, "gx");
        ObjectId gy = mid(ImageFormat::S16, "gy");
        ObjectId mag = image(ImageFormat::S16, "mag");
        g.add_node("Gaussian3x3", {cg.input, gs});
        g.add_node("Sobel3x3", {gs, gx, gy});
        g.add_node("Magnitude", {gx, gy, mag});
        cg.outputs = {mag};
        break;
    }
    case 2: {
        ObjectId gx = mid(ImageFormat::S16, "gx"), gy = mid(ImageFormat::S16, "gy");
        ObjectId ixx = mid(ImageFormat::S32, "ixx"), iyy = mid(ImageFormat::S32, "iyy"), ixy = mid(ImageFormat::S32, "ixy");
        ObjectId sxx = mid(ImageFormat::S32, "sxx"), syy = mid(ImageFormat::S32, "syy"), sxy = mid(ImageFormat::S32, "sxy");
        ObjectId resp = mid(ImageFormat::F32, "resp");
        ObjectId mask = image(ImageFormat::U8, "corners");
        g.add_node("Sobel3x3", {cg.input, gx, gy});
        g.add_node("Multiply", {gx, gx, ixx});
        g.add_node("Multiply", {gy, gy, iyy});
        g.add_node("Multiply", {gx, gy, ixy});
        g.add_node("Box3x3", {ixx, sxx});
        g.add_node("Box3x3", {iyy, syy});
        g.add_node("Box3x3", {ixy, sxy});
        g.add_node("HarrisResponse", {sxx, syy, sxy, resp});
        g.add_node("ThresholdF32", {resp, mask});
        cg.outputs = {mask};
        break;
    }
    case 3: {
        ObjectId blur = mid(ImageFormat::U8, "blur");
        ObjectId diff = mid(ImageFormat::S16, "diff");
        ObjectId sum = mid(ImageFormat::S16, "sum");
        ObjectId out = image(ImageFormat::U8, "sharp");
        g.add_node("Blur5x5", {cg.input, blur});
        g.add_node("Subtract", {cg.input, blur, diff});
        g.add_node("Add", {cg.input, diff, sum});
        g.add_node("ConvertDepth", {sum, out});
        cg.outputs = {out};
        break;
    }
    case 4: {
        std::vector<Value> m;
        for (std::int64_t v : binomial5()) m.push_back(Value::of_int(v));
        ObjectId mat = ctx.create_matrix(ScalarType::S32, 5, 5, m, "binomial5").id;
        g.note_data(mat);
        ObjectId conv = mid(ImageFormat::S16, "conv");
        ObjectId u8 = mid(ImageFormat::U8, "u8");
        ObjectId dist = ctx.create_array(ScalarType::S32, 256, "hist").id;
        ObjectId mean = ctx.create_scalar(ScalarType::F32, {}, "mean").id;
        ObjectId sd = ctx.create_scalar(ScalarType::F32, {}, "stddev").id;
        g.note_data(dist);
        g.note_data(mean);
        g.note_data(sd);
        g.add_node("Convolve", {cg.input, mat, conv}, {{"scale", std::int64_t{256}}});
        g.add_node("ConvertDepth", {conv, u8});
        g.add_node("Histogram", {u8, dist});
        g.add_node("MeanStdDev", {u8, mean, sd});
        cg.outputs = {dist, mean, sd};
        break;
    }
    default: throw std::runtime_error("unknown config " + std::to_string(cfg));
    }
    return cg;
}

/// verify -> expand -> verify: the implementation graph the executors run.
inline gvx::VerifiedGraph verified_impl(gvx::Context& ctx, const gvx::AppGraph& app) {
    gvx::VerifyResult vr = gvx::verify(app);
    if (!vr.ok()) throw std::runtime_error("config graph failed verification: " + vr.diagnostics.front().render());
    gvx::AppGraph& impl = gvx::expand(vr.verified, ctx);
    gvx::VerifyResult ir = gvx::verify(impl);
    if (!ir.ok()) throw std::runtime_error("implementation graph failed verification: " + ir.diagnostics.front().render());
    return ir.verified;
}

} // namespace gvx_configs
