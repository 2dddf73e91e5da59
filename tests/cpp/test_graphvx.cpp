// graphvx-b200 API and fusion tests (doctest stand-in).
//   CPU cases: object model fixes, DCE / transfer / fusion plans of the
//              BASELINE graphs, fusion refusal rules.
//   GPU cases (skipped without a CUDA device; the pytest wrapper runs them
//              under -m gpu): run_plan == run_naive bit-exactly on random
//              DAGs (SPEC.md:518 fusion soundness), custom kernels with every
//              boundary mode, device DivByZero, frame batches.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include "../../paper_2008_11476_b200/csrc/configs/config_graphs.hpp"
#include "graphvx/device.hpp"
#include "graphvx/image_io.hpp"
#include "graphvx/optimize.hpp"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <fstream>
#include <memory>
#include <random>
#include <tuple>

using namespace gvx;

namespace {

bool has_gpu() {
    static const int n = [] {
        if (std::getenv("GVX_TEST_CPU_ONLY")) return 0;
        return device_count();
    }();
    return n > 0;
}

#define GPU_ONLY()                                                                                                   \
    do {                                                                                                             \
        if (!has_gpu()) return;                                                                                      \
    } while (0)

ResolvedDesc img_desc(int w, int h, ImageFormat f) {
    ResolvedDesc d;
    d.kind = ObjKind::Image;
    d.width = w;
    d.height = h;
    d.format = f;
    return d;
}

VerifiedGraph impl_of(Context& ctx, const AppGraph& g) { return gvx_configs::verified_impl(ctx, g); }

bool same_outputs(const ExecutionReport& a, const ExecutionReport& b) {
    if (a.outputs.size() != b.outputs.size()) return false;
    for (const auto& [id, buf] : a.outputs) {
        auto it = b.outputs.find(id);
        if (it == b.outputs.end() || !buf.byte_equal(it->second)) return false;
    }
    return true;
}

} // namespace

// ----------------------------------------------------------------- CPU

TEST_CASE("virtual intermediates expand and fuse (reference CrossGraphVirtual defect fixed)") {
    for (int cfg : {1, 2, 3, 4}) {
        Context ctx;
        auto cg = gvx_configs::build_config(ctx, cfg, 64, 48, true);
        VerifiedGraph impl = impl_of(ctx, *cg.graph);
        CHECK(impl.stamped());
        OptimizedPlan plan = optimize(impl, ctx);
        CHECK(plan.fused.stamped());
        CHECK(plan.stats.launches_after <= plan.stats.launches_before);
    }
}

TEST_CASE("foreign virtual images are still rejected in application graphs") {
    Context ctx;
    AppGraph& g1 = ctx.create_graph();
    AppGraph& g2 = ctx.create_graph();
    ObjectId foreign = ctx.create_virtual_image(g1).id;
    ObjectId local = ctx.create_virtual_image(g2).id;
    CHECK_THROWS_AS(g2.add_node("Gaussian3x3", {foreign, local}), Error);
}

TEST_CASE("reference-granularity fusion of the BASELINE graphs (SURVEY.md 3.3)") {
    struct Want {
        int cfg, launches_after;
    };
    for (Want w : {Want{1, 3}, Want{2, 5}, Want{3, 1}, Want{4, 4}}) {
        Context ctx;
        auto cg = gvx_configs::build_config(ctx, w.cfg, 32, 32, true);
        OptimizedPlan plan = optimize(impl_of(ctx, *cg.graph), ctx);
        CAPTURE(w.cfg);
        CHECK(plan.stats.launches_after == w.launches_after);
        CHECK(plan.stats.nodes_removed == 0);
    }
}

TEST_CASE("transfer reduction: one upload and one download per graph input/output") {
    Context ctx;
    auto cg = gvx_configs::build_config(ctx, 1, 32, 32, true);
    OptimizedPlan plan = optimize(impl_of(ctx, *cg.graph), ctx);
    CHECK(plan.transfers.segment_count == 1);
    CHECK(plan.transfers.optimized_count() == 2);
    CHECK(plan.transfers.naive_count == 8);
}

TEST_CASE("dead computation elimination drops the unused Sobel half (paper Fig. 8 analogue)") {
    Context ctx;
    AppGraph& g = ctx.create_graph();
    ObjectId in = ctx.create_image(32, 32, ImageFormat::U8).id;
    ObjectId gx = ctx.create_image(32, 32, ImageFormat::S16).id;
    ObjectId gy = ctx.create_virtual_image(g).id;
    g.note_data(in);
    g.add_node("Sobel3x3", {in, gx, gy});
    OptimizedPlan plan = optimize(impl_of(ctx, g), ctx);
    CHECK(plan.stats.nodes_before == 2);
    CHECK(plan.stats.nodes_removed == 1);
}

namespace {
AbstractionPtr point_plus(int k) {
    std::vector<SignatureParam> ps(2);
    ps[0].direction = Direction::Input;
    ps[0].kind = ObjKind::Image;
    ps[1].direction = Direction::Output;
    ps[1].kind = ObjKind::Image;
    ps[1].formats = {ImageFormat::U8};
    PointKernel pk;
    pk.outputs.push_back(PointOutput{{saturate_to(ScalarType::U8, add(input_pixel(0), const_i(k)))}});
    return make_point_kernel("plus" + std::to_string(k), KernelSignature(ps), pk);
}

AbstractionPtr blur_local(BoundaryMode mode, std::int64_t constant) {
    std::vector<SignatureParam> ps(2);
    ps[0].direction = Direction::Input;
    ps[0].kind = ObjKind::Image;
    ps[1].direction = Direction::Output;
    ps[1].kind = ObjKind::Image;
    ps[1].formats = {ImageFormat::U8};
    LocalKernel lk;
    lk.window_w = 3;
    lk.window_h = 5;
    lk.boundary = mode;
    lk.boundary_value = Value::of_int(constant);
    lk.tap_body = window_pixel(0, 0, 0);
    lk.post_body = saturate_to(ScalarType::U8, div(add(input_pixel(0), const_i(7)), const_i(15)));
    return make_local_kernel(std::string("blur_") + to_string(mode), KernelSignature(ps), lk);
}

/// in -> plus3 -> blur(mode) -> plus5 -> out, all intermediates virtual.
struct Chain {
    Context ctx;
    AppGraph* g = nullptr;
    ObjectId in = 0, out = 0;
    explicit Chain(BoundaryMode mode, int w = 23, int h = 19) {
        auto reg = std::make_shared<KernelRegistry>(KernelRegistry::builtin().clone());
        reg->add_custom(point_plus(3));
        reg->add_custom(point_plus(5));
        reg->add_custom(blur_local(mode, 200));
        ctx.set_registry(reg);
        g = &ctx.create_graph();
        in = ctx.create_image(w, h, ImageFormat::U8).id;
        out = ctx.create_image(w, h, ImageFormat::U8).id;
        g->note_data(in);
        ObjectId a = ctx.create_virtual_image(*g).id, b = ctx.create_virtual_image(*g).id;
        g->add_node("plus3", {in, a});
        g->add_node(std::string("blur_") + to_string(mode), {a, b});
        g->add_node("plus5", {b, out});
    }
};
} // namespace

TEST_CASE("fusion refuses rewrites that would change results vs run_naive") {
    {
        Chain c(BoundaryMode::Clamp);
        OptimizedPlan p = optimize(impl_of(c.ctx, *c.g), c.ctx);
        CHECK(p.stats.launches_after == 1); // point->local->point fully fused under Clamp
    }
    {
        Chain c(BoundaryMode::Constant);
        OptimizedPlan p = optimize(impl_of(c.ctx, *c.g), c.ctx);
        CHECK(p.stats.launches_after == 2); // point->local refused (border constant)
    }
    {
        Chain c(BoundaryMode::Undefined);
        OptimizedPlan p = optimize(impl_of(c.ctx, *c.g), c.ctx);
        CHECK(p.stats.launches_after == 2); // local->point refused (border ring)
    }
}

TEST_CASE("execution without a device fails loudly (no host fallback)") {
    if (has_gpu()) return;
    Context ctx;
    auto cg = gvx_configs::build_config(ctx, 1, 16, 16, true);
    VerifiedGraph impl = impl_of(ctx, *cg.graph);
    InputMap in;
    in[cg.input] = random_buffer(img_desc(16, 16, ImageFormat::U8), 1);
    try {
        run_naive(impl, in);
        FAIL("expected UnsupportedKind");
    } catch (const Error& e) {
        CHECK(e.code() == ErrorCode::UnsupportedKind);
    }
}

TEST_CASE("image files: PGM / PPM / raw round trips and header errors (ref:src/image_io.cpp)") {
    const std::string dir = std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp";
    for (ImageFormat f : {ImageFormat::U8, ImageFormat::RGB, ImageFormat::S16, ImageFormat::F32, ImageFormat::UYVY}) {
        Buffer b = random_buffer(img_desc(37, 11, f), 5);
        const std::string path = dir + "/gvx_img_test" + default_extension(f);
        write_image_file(path, b);
        Buffer r = read_image_file(path);
        CHECK(r.desc.width == 37);
        CHECK(r.desc.height == 11);
        CHECK(r.desc.format == f);
        CHECK(r.bytes == b.bytes);
        std::remove(path.c_str());
    }
    CHECK(default_extension(ImageFormat::U8) == ".pgm");
    CHECK(default_extension(ImageFormat::RGB) == ".ppm");
    CHECK(default_extension(ImageFormat::S32) == ".raw");
    const std::string bad = dir + "/gvx_img_bad.pgm";
    {
        std::ofstream o(bad, std::ios::binary);
        o << "P5\n# comment\n4 2\n65535\n";
    }
    CHECK_THROWS_AS(read_image_file(bad), Error);
    {
        std::ofstream o(bad, std::ios::binary);
        o << "P5\n# comment\n4 2\n255\nab"; // truncated payload
    }
    CHECK_THROWS_AS(read_image_file(bad), Error);
    {
        std::ofstream o(bad, std::ios::binary);
        o << "P5 4 2 255\nabcdefgh"; // single-line header
    }
    Buffer ok = read_image_file(bad);
    CHECK(ok.desc.width == 4);
    CHECK(ok.bytes[7] == 'h');
    std::remove(bad.c_str());
    CHECK_THROWS_AS(read_image_file(dir + "/gvx_no_such_file.pgm"), Error);
}

// ----------------------------------------------------------------- GPU

TEST_CASE("gpu: boundary modes through fused plans equal run_naive") {
    GPU_ONLY();
    for (BoundaryMode m : {BoundaryMode::Clamp, BoundaryMode::Constant, BoundaryMode::Undefined}) {
        for (auto [w, h] : {std::pair{23, 19}, std::pair{1, 1}, std::pair{2, 7}, std::pair{200, 3}}) {
            Chain c(m, w, h);
            VerifiedGraph impl = impl_of(c.ctx, *c.g);
            OptimizedPlan p = optimize(impl, c.ctx);
            InputMap in;
            in[c.in] = random_buffer(img_desc(w, h, ImageFormat::U8), 99 + w);
            ExecutionReport a = run_naive(impl, in), b = run_plan(p, in);
            CAPTURE(to_string(m));
            CAPTURE(w);
            CHECK(same_outputs(a, b));
            CHECK(b.counters.kernel_launches <= a.counters.kernel_launches);
        }
    }
}

TEST_CASE("gpu: host API error contract of run_plan / run_naive (ref:src/execute.cpp:300-346, 880-897)") {
    GPU_ONLY();
    Context ctx;
    auto cg = gvx_configs::build_config(ctx, 1, 40, 30, true);
    VerifiedGraph impl = impl_of(ctx, *cg.graph);
    OptimizedPlan plan = optimize(impl, ctx);
    auto code_of = [](auto&& fn) {
        try {
            fn();
        } catch (const Error& e) {
            return static_cast<int>(e.code());
        }
        return -1;
    };
    const Buffer good = random_buffer(img_desc(40, 30, ImageFormat::U8), 3);
    for (bool naive : {false, true}) {
        auto run = [&](const InputMap& in) { return naive ? run_naive(impl, in) : run_plan(plan, in); };
        CAPTURE(naive);
        // MissingInput: a consumed input without a buffer (ref:src/execute.cpp:344)
        CHECK(code_of([&] { run(InputMap{}); }) == static_cast<int>(ErrorCode::MissingInput));
        // ShapeMismatch: declared 40x30 U8, got 41x30 / S16 (ref:src/execute.cpp:321)
        InputMap wrong;
        wrong[cg.input] = random_buffer(img_desc(41, 30, ImageFormat::U8), 3);
        CHECK(code_of([&] { run(wrong); }) == static_cast<int>(ErrorCode::ShapeMismatch));
        wrong[cg.input] = random_buffer(img_desc(40, 30, ImageFormat::S16), 3);
        CHECK(code_of([&] { run(wrong); }) == static_cast<int>(ErrorCode::ShapeMismatch));
        // UnknownObject: a buffer for an id the context does not know (ref:src/execute.cpp:304)
        InputMap unknown;
        unknown[cg.input] = good;
        unknown[987654] = good;
        CHECK(code_of([&] { run(unknown); }) == static_cast<int>(ErrorCode::UnknownObject));
        // AccessDenied: writing a virtual intermediate from the host (ref:src/execute.cpp:306)
        ObjectId virt = kInvalidId;
        for (ObjectId id : cg.graph->data())
            if (ctx.find(id) && ctx.find(id)->is_virtual) virt = id;
        REQUIRE(virt != kInvalidId);
        InputMap denied;
        denied[cg.input] = good;
        denied[virt] = good;
        CHECK(code_of([&] { run(denied); }) == static_cast<int>(ErrorCode::AccessDenied));
        // the good run still works after every failure (no poisoned device state)
        InputMap ok;
        ok[cg.input] = good;
        CHECK(run(ok).outputs.size() == 1);
    }
    // UnstampedGraph: an unverified graph / plan (ref:src/execute.cpp:881, 891)
    VerifiedGraph blank;
    OptimizedPlan blank_plan;
    InputMap ok;
    ok[cg.input] = good;
    CHECK(code_of([&] { run_naive(blank, ok); }) == static_cast<int>(ErrorCode::UnstampedGraph));
    CHECK(code_of([&] { run_plan(blank_plan, ok); }) == static_cast<int>(ErrorCode::UnstampedGraph));
}

TEST_CASE("gpu: row bands of a mixed program (generated + hand-written units) equal run_plan") {
    GPU_ONLY();
    // Dilate -> Median -> AbsDiff(in) -> Sobel -> Magnitude -> ConvertDepth:
    // generated local / point kernels and the fused edge group, with
    // intermediates in HBM between units and halos of 1 row per local
    for (auto [w, h, nb] : {std::tuple{200, 97, 3}, std::tuple{64, 40, 5}, std::tuple{131, 23, 2}}) {
        Context ctx;
        AppGraph& g = ctx.create_graph();
        auto img = [&](ImageFormat f, bool virt) {
            if (virt) return ctx.create_virtual_image(g).id; // format / size inferred by verify
            ObjectId id = ctx.create_image(w, h, f).id;
            g.note_data(id);
            return id;
        };
        const ObjectId in = img(ImageFormat::U8, false), a = img(ImageFormat::U8, true), b = img(ImageFormat::U8, true);
        const ObjectId c = img(ImageFormat::U8, true), gx = img(ImageFormat::S16, true), gy = img(ImageFormat::S16, true);
        const ObjectId mag = img(ImageFormat::S16, true), out = img(ImageFormat::U8, false);
        g.add_node("Dilate3x3", {in, a});
        g.add_node("Median3x3", {a, b});
        g.add_node("AbsDiff", {b, in, c});
        g.add_node("Sobel3x3", {c, gx, gy});
        g.add_node("Magnitude", {gx, gy, mag});
        AttrMap at;
        at["shift"] = std::int64_t{2};
        g.add_node("ConvertDepth", {mag, out}, at);
        VerifiedGraph impl = impl_of(ctx, g);
        OptimizedPlan plan = optimize(impl, ctx);
        InputMap inputs;
        inputs[in] = random_buffer(img_desc(w, h, ImageFormat::U8), 5 + w);
        const ExecutionReport want = run_plan(plan, inputs);
        std::unique_ptr<BandGroup> grp_p;
        try {
            grp_p = std::make_unique<BandGroup>(plan, std::vector<int>(static_cast<std::size_t>(nb), 0));
        } catch (const std::exception& e) {
            FAIL(std::string("BandGroup construction: ") + e.what() + "\n" + DeviceSession(plan).describe());
        }
        BandGroup& grp = *grp_p;
        std::vector<std::uint8_t> got(static_cast<std::size_t>(w) * h, 0xEE);
        for (int k = 0; k < nb; ++k) {
            const BandLayout L = grp.band(k).layout();
            grp.band(k).upload_rows(in, inputs[in].bytes.data() + static_cast<std::size_t>(L.row0) * w, w, L.row0,
                                    L.row1 - L.row0);
        }
        try {
            grp.launch();
            grp.synchronize();
        } catch (const std::exception& e) {
            FAIL(std::string("BandGroup launch: ") + e.what() + "\n" + DeviceSession(plan).describe());
        }
        for (int k = 0; k < nb; ++k) {
            const BandLayout L = grp.band(k).layout();
            grp.band(k).download_rows(out, got.data() + static_cast<std::size_t>(L.row0) * w, w, L.row0,
                                      L.row1 - L.row0);
        }
        CAPTURE(w);
        CAPTURE(nb);
        CHECK(grp.band(0).describe().find("nvrtc") != std::string::npos);
        CHECK(got == want.outputs.at(out).bytes);
    }
}

TEST_CASE("gpu: DivByZero and results through the row-piece host path") {
    GPU_ONLY();
    // one input, one group, a 1 MB frame: run_naive / run_plan take the
    // pipelined row-piece path (execute.cpp host_piece_rows)
    std::vector<SignatureParam> ps(2);
    ps[0].direction = Direction::Input;
    ps[0].kind = ObjKind::Image;
    ps[1].direction = Direction::Output;
    ps[1].kind = ObjKind::Image;
    ps[1].formats = {ImageFormat::U8};
    PointKernel pk;
    pk.arity = 1;
    pk.outputs.push_back(PointOutput{{saturate_to(ScalarType::U8, div(const_i(1000), input_pixel(0)))}});
    auto reg = std::make_shared<KernelRegistry>(KernelRegistry::builtin().clone());
    reg->add_custom(make_point_kernel("inverse", KernelSignature(ps), pk));
    Context ctx;
    ctx.set_registry(reg);
    AppGraph& g = ctx.create_graph();
    const int W = 1024, H = 1031;
    ObjectId a = ctx.create_image(W, H, ImageFormat::U8).id, o = ctx.create_image(W, H, ImageFormat::U8).id;
    g.note_data(a);
    g.add_node("inverse", {a, o});
    VerifiedGraph impl = impl_of(ctx, g);
    InputMap ok, bad;
    ok[a] = random_buffer(img_desc(W, H, ImageFormat::U8), 4);
    for (auto& v : ok[a].bytes) v |= 1;
    bad = ok;
    bad[a].bytes[static_cast<std::size_t>(W) * (H - 3) + 17] = 0; // in the last piece
    const ExecutionReport r1 = run_naive(impl, ok);
    bool raised = false;
    try {
        run_naive(impl, bad);
    } catch (const Error& e) {
        raised = e.code() == ErrorCode::DivByZero;
    }
    CHECK(raised);
    const ExecutionReport r2 = run_naive(impl, ok); // the status was cleared
    CHECK(r2.outputs.at(o).bytes == r1.outputs.at(o).bytes);
    const auto& in = ok[a].bytes;
    const auto& out = r1.outputs.at(o).bytes;
    bool exact = out.size() == in.size();
    for (std::size_t i = 0; exact && i < in.size(); ++i) exact = out[i] == std::min(255, 1000 / in[i]);
    CHECK(exact);
}

TEST_CASE("gpu: runtime division by zero surfaces as DivByZero") {
    GPU_ONLY();
    std::vector<SignatureParam> ps(3);
    ps[0].direction = ps[1].direction = Direction::Input;
    ps[0].kind = ps[1].kind = ObjKind::Image;
    ps[2].direction = Direction::Output;
    ps[2].kind = ObjKind::Image;
    ps[2].formats = {ImageFormat::U8};
    PointKernel pk;
    pk.arity = 2;
    pk.outputs.push_back(PointOutput{{saturate_to(ScalarType::U8, div(input_pixel(0), input_pixel(1)))}});
    auto reg = std::make_shared<KernelRegistry>(KernelRegistry::builtin().clone());
    reg->add_custom(make_point_kernel("ratio", KernelSignature(ps), pk));
    Context ctx;
    ctx.set_registry(reg);
    AppGraph& g = ctx.create_graph();
    ObjectId a = ctx.create_image(8, 8, ImageFormat::U8).id, b = ctx.create_image(8, 8, ImageFormat::U8).id;
    ObjectId o = ctx.create_image(8, 8, ImageFormat::U8).id;
    g.note_data(a);
    g.note_data(b);
    g.add_node("ratio", {a, b, o});
    VerifiedGraph impl = impl_of(ctx, g);
    InputMap in;
    in[a] = random_buffer(img_desc(8, 8, ImageFormat::U8), 1);
    in[b] = Buffer::image(img_desc(8, 8, ImageFormat::U8)); // zeros
    CHECK_THROWS_AS(run_naive(impl, in), Error);
    try {
        run_naive(impl, in);
    } catch (const Error& e) {
        CHECK(e.code() == ErrorCode::DivByZero);
    }
    // the pipelined host path reports it for the offending frame only
    HostPipeline pipe(impl, 2);
    InputMap ok = in;
    ok[b] = random_buffer(img_desc(8, 8, ImageFormat::U8), 2);
    for (std::size_t i = 0; i < ok[b].bytes.size(); ++i) ok[b].bytes[i] |= 1; // no zero divisor
    pipe.submit(ok);
    pipe.submit(in);
    ExecutionReport first = pipe.next();
    CHECK(first.outputs.at(o).bytes == run_naive(impl, ok).outputs.at(o).bytes);
    bool raised = false;
    try {
        pipe.next();
    } catch (const Error& e) {
        raised = e.code() == ErrorCode::DivByZero;
    }
    CHECK(raised);
    pipe.submit(ok); // the pipeline stays usable
    CHECK(pipe.next().outputs.at(o).bytes == first.outputs.at(o).bytes);

    // concurrent executions keep their own error flags and counters: a
    // thread hitting DivByZero never leaks it into another graph's run
    Context ctx2;
    gvx_configs::ConfigGraph cg = gvx_configs::build_config(ctx2, 2, 97, 61, true);
    VerifiedGraph impl2 = impl_of(ctx2, *cg.graph);
    OptimizedPlan plan2 = optimize(impl2, ctx2);
    InputMap in2;
    in2[cg.input] = random_buffer(img_desc(97, 61, ImageFormat::U8), 3);
    const ExecutionReport want = run_plan(plan2, in2);
    std::atomic<int> bad{0}, div_errors{0};
    std::thread t1([&] {
        for (int i = 0; i < 40; ++i) {
            try {
                run_naive(impl, in);
            } catch (const Error& e) {
                if (e.code() == ErrorCode::DivByZero) ++div_errors;
            }
        }
    });
    std::thread t2([&] {
        for (int i = 0; i < 40; ++i) {
            try {
                const ExecutionReport r = run_plan(plan2, in2);
                if (!same_outputs(r, want) || r.counters.pixels_read != want.counters.pixels_read) ++bad;
            } catch (const Error&) {
                ++bad;
            }
        }
    });
    t1.join();
    t2.join();
    CHECK(bad.load() == 0);
    CHECK(div_errors.load() == 40);
}

namespace {

/// Random DAG over the registry (point, local, global kinds).
struct RandomGraph {
    Context ctx;
    AppGraph* g = nullptr;
    std::vector<ObjectId> inputs;
    RandomGraph(std::uint64_t seed, int w, int h) {
        std::mt19937_64 rng(seed);
        g = &ctx.create_graph();
        std::vector<ObjectId> u8, s16;
        for (int i = 0; i < 2; ++i) {
            ObjectId id = ctx.create_image(w, h, ImageFormat::U8).id;
            g->note_data(id);
            inputs.push_back(id);
            u8.push_back(id);
        }
        auto pick = [&](std::vector<ObjectId>& v) { return v[rng() % v.size()]; };
        auto fresh = [&](ImageFormat f, bool last) {
            const bool virt = !last && (rng() % 10) < 7;
            ObjectId id = virt ? ctx.create_virtual_image(*g).id : ctx.create_image(w, h, f).id;
            g->note_data(id);
            return id;
        };
        const int n = 3 + static_cast<int>(rng() % 6);
        for (int i = 0; i < n; ++i) {
            const bool last = i == n - 1;
            switch (rng() % 11) {
            case 0: { ObjectId o = fresh(ImageFormat::U8, last); g->add_node("Gaussian3x3", {pick(u8), o}); u8.push_back(o); break; }
            case 1: { ObjectId o = fresh(ImageFormat::U8, last); g->add_node("Box3x3", {pick(u8), o}); u8.push_back(o); break; }
            case 2: { ObjectId x = fresh(ImageFormat::S16, last), y = fresh(ImageFormat::S16, last);
                      g->add_node("Sobel3x3", {pick(u8), x, y}); s16.push_back(x); s16.push_back(y); break; }
            case 3: { ObjectId o = fresh(ImageFormat::U8, last); g->add_node("Dilate3x3", {pick(u8), o}); u8.push_back(o); break; }
            case 4: { ObjectId o = fresh(ImageFormat::U8, last); g->add_node("Median3x3", {pick(u8), o}); u8.push_back(o); break; }
            case 5: { ObjectId o = fresh(ImageFormat::S16, last); g->add_node("Subtract", {pick(u8), pick(u8), o}); s16.push_back(o); break; }
            case 6: { if (s16.size() < 2) { --i; break; }
                      ObjectId o = fresh(ImageFormat::S16, last); g->add_node("Magnitude", {pick(s16), pick(s16), o}); s16.push_back(o); break; }
            case 7: { if (s16.empty()) { --i; break; }
                      ObjectId o = fresh(ImageFormat::U8, last); g->add_node("ConvertDepth", {pick(s16), o}); u8.push_back(o); break; }
            case 8: { ObjectId o = fresh(ImageFormat::U8, last); g->add_node("AbsDiff", {pick(u8), pick(u8), o}); u8.push_back(o); break; }
            case 9: { ObjectId t = ctx.create_scalar(ScalarType::U8, Value::of_int(static_cast<std::int64_t>(rng() % 256))).id;
                      g->note_data(t);
                      ObjectId o = fresh(ImageFormat::U8, last); g->add_node("Threshold", {pick(u8), t, kInvalidId, o}); u8.push_back(o); break; }
            default: { ObjectId o = fresh(ImageFormat::U8, last); g->add_node("Not", {pick(u8), o}); u8.push_back(o); break; }
            }
        }
    }
};

} // namespace

TEST_CASE("gpu: fusion soundness on random DAGs (run_plan == run_naive, bit exact)") {
    GPU_ONLY();
    int checked = 0;
    // 100 graphs: local -> local pairs with virtual intermediates (the generic
    // on-chip chains) appear in most of them
    for (std::uint64_t seed = 1; seed <= 100; ++seed) {
        const int w = 5 + static_cast<int>(seed * 37 % 120), h = 3 + static_cast<int>(seed * 11 % 50);
        RandomGraph rg(seed, w, h);
        VerifyResult vr = verify(*rg.g);
        if (!vr.ok()) continue;
        VerifiedGraph impl = impl_of(rg.ctx, *rg.g);
        OptimizedPlan plan = optimize(impl, rg.ctx);
        InputMap in;
        for (ObjectId id : rg.inputs) in[id] = random_buffer(img_desc(w, h, ImageFormat::U8), seed * 3 + id);
        ExecutionReport a = run_naive(impl, in);
        ExecutionReport b = run_plan(plan, in);
        CAPTURE(seed);
        CHECK(same_outputs(a, b));
        CHECK(b.counters.kernel_launches <= a.counters.kernel_launches);
        CHECK(b.counters.transfers_executed <= a.counters.transfers_executed);
        ++checked;
    }
    CHECK(checked >= 75);
}

TEST_CASE("gpu: frame batches through a DeviceSession equal per-frame run_plan") {
    GPU_ONLY();
    for (int cfg : {1, 2, 3, 4}) {
        Context ctx;
        auto cg = gvx_configs::build_config(ctx, cfg, 77, 41, true);
        OptimizedPlan plan = optimize(impl_of(ctx, *cg.graph), ctx);
        const int frames = 3;
        DeviceSession s(plan, frames);
        std::vector<Buffer> ins;
        for (int f = 0; f < frames; ++f) {
            ins.push_back(random_buffer(img_desc(77, 41, ImageFormat::U8), 500 + f));
            s.upload(cg.input, ins.back(), f);
        }
        s.launch();
        s.synchronize();
        for (int f = 0; f < frames; ++f) {
            InputMap in;
            in[cg.input] = ins[static_cast<std::size_t>(f)];
            ExecutionReport r = run_plan(plan, in);
            for (ObjectId o : cg.outputs) {
                CAPTURE(cfg);
                CAPTURE(f);
                CHECK(s.download(o, f).byte_equal(r.outputs.at(o)));
            }
        }
    }
}
