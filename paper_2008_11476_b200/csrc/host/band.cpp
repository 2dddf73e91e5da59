// Row-band execution of an optimized plan over several GPUs (device.hpp:
// BandedSession, BandGroup).  No reference counterpart: the reference
// splits rows over <= 4 host threads of one process
// (ref:src/execute.cpp:392-419); here each band is a GPU, one halo exchange
// per fused stencil group, all device work through the
// C-ABI (include/gvxb.h).
//
// Storage: every image object of the program is held as a slab of global
// rows [row0 - R, row1 + R) clipped to the image, R = the largest radius of
// the groups reading it (0 for outputs).  A group's launch writes rows
// [row0, row1) of its outputs; before it runs, the R rows of its input that
// the band does not own are received from the neighbours (the interior rows
// run meanwhile: they read owned rows only).
#include "graphvx/device.hpp"
#include "graphvx/error.hpp"
#include "hostcopy.hpp"
#include "program.hpp"

#include <algorithm>
#include <cstring>
#include <set>
#include <sstream>

namespace gvx {

namespace {

using dev::check;

/// Image inputs of a unit with the rows beyond its output rows it reads
/// them at, or false when the unit cannot run on a row band.
bool band_inputs(const dev::Unit& u, const std::map<ObjectId, dev::ObjInfo>& objects,
                 std::vector<std::pair<ObjectId, int>>& out) {
    out.clear();
    switch (u.kind) {
    case dev::Unit::Kind::Edge: out.push_back({u.src, u.with_gauss ? 2 : 1}); return true; // Gaussian + Sobel
    case dev::Unit::Kind::Harris: out.push_back({u.src, 2}); return true;                  // Sobel + Box3x3
    case dev::Unit::Kind::Stencil: out.push_back({u.src, u.ksize / 2}); return true;
    case dev::Unit::Kind::Jit: {
        if (u.prog.in_halo.size() != u.in_ids.size()) return false; // global ops, scans, scaling
        for (const jit::KernelSpec& ks : u.prog.kernels)
            if (ks.grid != jit::KernelSpec::Grid::Pixels && ks.grid != jit::KernelSpec::Grid::OutPixels) return false;
        for (std::size_t i = 0; i < u.in_ids.size(); ++i) {
            const ObjectId id = u.in_ids[i];
            if (id == kInvalidId) continue;
            auto it = objects.find(id);
            if (it == objects.end()) continue;
            if (it->second.desc.kind == ObjKind::Image) out.push_back({id, u.prog.in_halo[i]});
            else if (it->second.desc.kind != ObjKind::Matrix) return false; // run-time scalars / arrays
        }
        return true;
    }
    default: return false;
    }
}

int unit_halo(const std::vector<std::pair<ObjectId, int>>& ins) {
    int r = 0;
    for (const auto& kv : ins) r = std::max(r, kv.second);
    return r;
}

struct Slab {
    void* ptr = nullptr;
    std::int64_t pitch = 0, fstride = 0;
    int row0 = 0, rows = 0; ///< global rows held
    int halo = 0;           ///< rows beyond the band on each side (clipped)
    int bpp = 1, format = 0;
    bool owned = false;
};

} // namespace

struct BandedSession::Impl {
    std::shared_ptr<dev::Program> prog;
    int rank = 0, world = 1, device = 0, frames = 1;
    int W = 0, H = 0;
    gvxb_ctx ctx = nullptr;  ///< compute stream
    gvxb_ctx xctx = nullptr; ///< exchange stream (peer copies in a group)
    gvxb_comm comm = nullptr;
    gvxb_band_plan band{};   ///< rows of this band (halo 0)
    std::map<ObjectId, Slab> slabs;
    std::vector<gvxb_band_plan> unit_plan; ///< per unit: split by its largest input halo
    std::vector<std::vector<std::pair<ObjectId, int>>> unit_ins; ///< per unit: image inputs and halos
    std::map<ObjectId, gvxb_band_plan> obj_plan;  ///< exchange of an object's whole slab halo
    std::set<ObjectId> exchanged;                 ///< objects exchanged in the current launch
    int input_halo = 0;
    ObjectId input = kInvalidId;

    // BandGroup wiring (peer copies)
    std::vector<Impl*>* group = nullptr;
    int index = 0;
    void* ev_ready = nullptr; ///< compute stream reached the exchange point
    void* ev_xdone = nullptr; ///< exchange stream finished pulling
    bool pulled = false;

    // run_host pipeline
    gvxb_ctx up = nullptr, dn = nullptr;
    std::vector<void*> ev_up, ev_k;

    ~Impl() {
        if (ctx) gvxb_sync(ctx);
        if (xctx) gvxb_sync(xctx);
        if (up) gvxb_sync(up);
        if (dn) gvxb_sync(dn);
        for (auto& kv : slabs)
            if (kv.second.owned) gvxb_free(ctx, kv.second.ptr);
        for (void* e : ev_up) gvxb_event_destroy(e);
        for (void* e : ev_k) gvxb_event_destroy(e);
        for (void* e : ev_dn) gvxb_event_destroy(e);
        for (void* e : ev_in_free) gvxb_event_destroy(e);
        for (void* q : stage_in) gvxb_host_free(q);
        for (void* q : stage_out) gvxb_host_free(q);
        if (ev_ready) gvxb_event_destroy(ev_ready);
        if (ev_xdone) gvxb_event_destroy(ev_xdone);
        for (gvxb_ctx c : {up, dn, xctx, ctx})
            if (c) gvxb_ctx_destroy(c);
    }

    void init(const OptimizedPlan& plan, int rank_, int world_, void* comm_, int device_, int frames_) {
        init_program(dev::program_of(plan), rank_, world_, comm_, device_, frames_);
    }

    void init_program(std::shared_ptr<dev::Program> prog_, int rank_, int world_, void* comm_, int device_,
                      int frames_) {
        prog = std::move(prog_);
        rank = rank_;
        world = world_;
        frames = std::max(1, frames_);
        comm = static_cast<gvxb_comm>(comm_);
        if (world < 1 || rank < 0 || rank >= world) throw Error(ErrorCode::BadKernel, "bad band rank / world");
        std::map<ObjectId, int> radius_in; // object -> largest halo of the units reading it
        for (const dev::Unit& u : prog->units) {
            std::vector<std::pair<ObjectId, int>> ins;
            if (!band_inputs(u, prog->objects, ins))
                throw Error(ErrorCode::UnsupportedKind,
                            "row-band execution needs stencil / point programs; '" + u.label +
                                "' is a global operation or reads run-time scalars (run it with DeviceSession per frame "
                                "instead)");
            for (const auto& [id, r] : ins) radius_in[id] = std::max(radius_in[id], r);
            unit_ins.push_back(std::move(ins));
        }
        if (prog->units.empty()) throw Error(ErrorCode::UnsupportedKind, "row-band execution of an empty program");
        for (const auto& [id, oi] : prog->objects) {
            if (oi.desc.kind == ObjKind::Matrix) continue; // baked into the generated code
            if (oi.desc.kind != ObjKind::Image)
                throw Error(ErrorCode::UnsupportedKind, "row-band execution: non-image object in the program", id);
            if (W == 0) W = oi.desc.width, H = oi.desc.height;
            if (oi.desc.width != W || oi.desc.height != H)
                throw Error(ErrorCode::UnsupportedKind, "row-band execution needs images of one size", id);
        }
        device = device_ >= 0 ? device_ : gvxb_ctx_device(dev::context());
        ctx = dev::own_context(device);
        check(gvxb_band_plan_make(H, world, rank, 0, &band), "band plan");
        for (const auto& [id, oi] : prog->objects) {
            if (oi.desc.kind != ObjKind::Image) continue;
            auto it = radius_in.find(id);
            const int R = it == radius_in.end() ? 0 : it->second;
            gvxb_band_plan p{};
            check(gvxb_band_plan_make(H, world, rank, R, &p), "band plan");
            Slab s;
            s.row0 = p.src_row0;
            s.rows = p.src_row1 - p.src_row0;
            s.halo = R;
            s.bpp = bytes_per_pixel(oi.desc.format);
            s.format = static_cast<int>(oi.desc.format);
            const std::int64_t row = static_cast<std::int64_t>(W) * s.bpp;
            s.pitch = std::max<std::int64_t>(128, (row + 127) / 128 * 128);
            s.fstride = s.pitch * std::max(1, s.rows);
            s.owned = true;
            const std::size_t bytes = static_cast<std::size_t>(s.fstride) * frames;
            check(gvxb_alloc(ctx, bytes, &s.ptr), "band allocation");
            check(gvxb_memset(ctx, s.ptr, 0, bytes), "band clear");
            slabs[id] = s;
            if (!oi.produced && R > 0 && input == kInvalidId) input = id, input_halo = R;
        }
        if (input == kInvalidId && !unit_ins.front().empty())
            input = unit_ins.front().front().first, input_halo = radius_in[input];
        for (std::size_t i = 0; i < prog->units.size(); ++i) {
            gvxb_band_plan p{};
            check(gvxb_band_plan_make(H, world, rank, unit_halo(unit_ins[i]), &p), "band plan");
            unit_plan.push_back(p);
            for (const auto& kv : unit_ins[i]) {
                if (obj_plan.count(kv.first)) continue;
                gvxb_band_plan q{};
                check(gvxb_band_plan_make(H, world, rank, slabs.at(kv.first).halo, &q), "band plan");
                obj_plan[kv.first] = q;
            }
        }
    }

    gvxb_image image(ObjectId id, bool at_band_row0) {
        gvxb_image im{};
        if (id == kInvalidId) return im;
        const Slab& s = slabs.at(id);
        const int skip = at_band_row0 ? band.row0 - s.row0 : 0;
        im.data = static_cast<char*>(s.ptr) + static_cast<std::int64_t>(skip) * s.pitch;
        im.pitch = s.pitch;
        im.width = W;
        im.height = s.rows - skip;
        im.format = s.format;
        im.frames = frames;
        im.frame_stride = s.fstride;
        return im;
    }

    /// Output rows [r0, r1) of unit `u` (its input halo rows must be present).
    void compute(const dev::Unit& u, int r0, int r1, gvxb_ctx on) {
        if (r1 <= r0) return;
        if (u.kind == dev::Unit::Kind::Jit) {
            compute_jit(u, r0, r1, on);
            return;
        }
        const Slab& src = slabs.at(u.src);
        const gvxb_band b{r0, r1, H, src.row0, band.row0};
        switch (u.kind) {
        case dev::Unit::Kind::Edge: {
            gvxb_edge_args a{};
            a.src = image(u.src, false);
            a.gx = image(u.out[0], true);
            a.gy = image(u.out[1], true);
            a.mag = image(u.out[2], true);
            a.with_gauss = u.with_gauss ? 1 : 0;
            a.band = b;
            check(gvxb_edge(on, &a), "gvxb_edge (band)");
            return;
        }
        case dev::Unit::Kind::Harris: {
            gvxb_harris_args a{};
            a.src = image(u.src, false);
            a.mask = image(u.out[0], true);
            a.response = image(u.out[1], true);
            a.k = u.k_param;
            a.threshold = u.threshold;
            a.band = b;
            check(gvxb_harris(on, &a), "gvxb_harris (band)");
            return;
        }
        case dev::Unit::Kind::Stencil: {
            gvxb_stencil_args a{};
            a.src = image(u.src, false);
            a.dst = image(u.out[0], true);
            a.ksize = u.ksize;
            std::memcpy(a.mask, u.mask, sizeof(a.mask));
            a.div_num = 1;
            a.div_den = u.divisor;
            a.mode = u.mode;
            a.band = b;
            check(gvxb_stencil_point(on, &a), "gvxb_stencil_point (band)");
            return;
        }
        case dev::Unit::Kind::Jit: compute_jit(u, r0, r1, on); return;
        default: throw Error(ErrorCode::UnsupportedKind, "row-band execution: unsupported group");
        }
    }

    /// A generated kernel set on output rows [r0, r1): image slots get the
    /// address of their global row 0 inside the slab (rows outside the slab
    /// are never read: its halo covers the kernel's windows).
    void compute_jit(const dev::Unit& u, int r0, int r1, gvxb_ctx on) {
        const jit::NodeProgram& np = u.prog;
        std::vector<std::uint64_t> f(static_cast<std::size_t>(np.fields()), 0);
        unsigned long long* counter = nullptr;
        std::uint32_t* status = nullptr;
        gvxb_counter_ptr(on, &counter);
        gvxb_status_ptr(on, &status);
        f[0] = reinterpret_cast<std::uint64_t>(status);
        f[1] = reinterpret_cast<std::uint64_t>(counter);
        f[2] = static_cast<std::uint64_t>(W);
        f[3] = static_cast<std::uint64_t>(H);
        f[4] = static_cast<std::uint64_t>(frames);
        auto put = [&](int slot, ObjectId id) {
            if (id == kInvalidId) return;
            auto it = slabs.find(id);
            if (it == slabs.end()) return; // matrices: baked into the code
            const Slab& sl = it->second;
            const std::size_t b = static_cast<std::size_t>(5 + 3 * slot);
            f[b] = reinterpret_cast<std::uint64_t>(static_cast<char*>(sl.ptr) - static_cast<std::int64_t>(sl.row0) * sl.pitch);
            f[b + 1] = static_cast<std::uint64_t>(sl.pitch);
            f[b + 2] = static_cast<std::uint64_t>(sl.fstride);
        };
        for (std::size_t i = 0; i < u.in_ids.size(); ++i) put(static_cast<int>(i), u.in_ids[i]);
        for (std::size_t o = 0; o < u.out_ids.size(); ++o) put(static_cast<int>(u.in_ids.size() + o), u.out_ids[o]);
        f[f.size() - 4] = static_cast<std::uint64_t>(r0);
        f[f.size() - 3] = static_cast<std::uint64_t>(r1);
        void* args[] = {f.data()};
        for (std::size_t ki = 0; ki < np.kernels.size(); ++ki) {
            const jit::KernelSpec& ks = np.kernels[ki];
            const unsigned grid[3] = {static_cast<unsigned>((W + ks.block_x * ks.cols - 1) / (ks.block_x * ks.cols)),
                                      static_cast<unsigned>((r1 - r0 + ks.block_y * ks.rows - 1) / (ks.block_y * ks.rows)),
                                      static_cast<unsigned>(frames)};
            const unsigned block[3] = {static_cast<unsigned>(ks.block_x), static_cast<unsigned>(ks.block_y), 1};
            check(gvxb_jit_launch(on, u.module, static_cast<int>(ki), grid, block, 0, args), "generated kernel (band)");
        }
    }

    /// Inputs of unit i whose halo rows must come from the neighbours (not
    /// yet exchanged in this launch).
    std::vector<ObjectId> pending_exchange(std::size_t i) const {
        std::vector<ObjectId> v;
        if (world <= 1) return v;
        for (const auto& kv : unit_ins[i]) {
            const gvxb_band_plan& q = obj_plan.at(kv.first);
            if ((q.peer[0] >= 0 || q.peer[1] >= 0) && !exchanged.count(kv.first)) v.push_back(kv.first);
        }
        return v;
    }
    bool needs_exchange(std::size_t i) const { return !pending_exchange(i).empty(); }
    /// Whether unit i's inputs have halo rows from neighbours at all.
    bool has_exchange(std::size_t i) const {
        if (world <= 1) return false;
        for (const auto& kv : unit_ins[i]) {
            const gvxb_band_plan& q = obj_plan.at(kv.first);
            if (q.peer[0] >= 0 || q.peer[1] >= 0) return true;
        }
        return false;
    }

    /// Posts the halo exchange of unit i's inputs (NCCL).  Peer mode: BandGroup.
    void exchange_nccl(std::size_t i) {
        if (!comm) throw Error(ErrorCode::UnsupportedKind, "row bands with world > 1 need a communicator or a BandGroup");
        for (ObjectId id : pending_exchange(i)) {
            gvxb_image slab = image(id, false);
            check(gvxb_halo_start(ctx, comm, &obj_plan.at(id), &slab), "halo exchange");
            exchanged.insert(id);
        }
    }

    /// Peer mode, phase 2: pull unit i's inputs' halo rows from the neighbours
    /// on the exchange stream once both sides reached the exchange point.
    void exchange_peer(std::size_t i) {
        check(gvxb_stream_wait_event(xctx, ev_ready), "exchange ordering");
        for (ObjectId id : pending_exchange(i)) {
            exchange_peer_object(id);
            exchanged.insert(id);
        }
        check(gvxb_event_record(xctx, ev_xdone), "exchange event");
        pulled = true;
    }

    void exchange_peer_object(ObjectId id) {
        const gvxb_band_plan& q = obj_plan.at(id);
        const Slab& me = slabs.at(id);
        for (int side = 0; side < 2; ++side) {
            if (q.peer[side] < 0) continue;
            Impl* nb = (*group)[static_cast<std::size_t>(q.peer[side])];
            check(gvxb_stream_wait_event(xctx, nb->ev_ready), "exchange ordering");
            const Slab& ns = nb->slabs.at(id);
            for (int f = 0; f < frames; ++f) {
                char* dst = static_cast<char*>(me.ptr) + f * me.fstride +
                            static_cast<std::int64_t>(q.recv_row0[side] - me.row0) * me.pitch;
                const char* src = static_cast<const char*>(ns.ptr) + f * ns.fstride +
                                  static_cast<std::int64_t>(q.recv_row0[side] - ns.row0) * ns.pitch;
                check(gvxb_copy_peer_rows(xctx, dst, static_cast<std::size_t>(me.pitch), device, src,
                                          static_cast<std::size_t>(ns.pitch), nb->device,
                                          static_cast<std::size_t>(W) * me.bpp,
                                          static_cast<std::size_t>(q.recv_rows[side])),
                      "halo peer copy");
            }
        }
    }

    void wait_exchange() {
        if (group) check(gvxb_stream_wait_event(ctx, ev_xdone), "halo wait");
        else check(gvxb_halo_wait(ctx, comm), "halo wait");
    }

    /// Unit i after its exchange was posted: interior rows, wait, edge rows.
    void run_unit(std::size_t i, bool exchanged) {
        const dev::Unit& u = prog->units[i];
        if (!exchanged) {
            compute(u, band.row0, band.row1, ctx);
            return;
        }
        const gvxb_band_plan& p = unit_plan[i];
        compute(u, p.interior_row0, p.interior_row1, ctx);
        wait_exchange();
        for (int e = 0; e < p.n_edges; ++e) compute(u, p.edge_row0[e], p.edge_row1[e], ctx);
    }

    void launch_standalone() {
        exchanged.clear();
        for (std::size_t i = 0; i < prog->units.size(); ++i) {
            const bool x = needs_exchange(i);
            if (x) exchange_nccl(i);
            run_unit(i, x);
        }
    }

    void ensure_pipeline(std::size_t pieces) {
        if (!up) up = dev::own_context(device), dn = dev::own_context(device);
        while (ev_up.size() < pieces) {
            void* a = nullptr;
            void* b = nullptr;
            check(gvxb_event_create(&a), "event");
            check(gvxb_event_create(&b), "event");
            ev_up.push_back(a);
            ev_k.push_back(b);
        }
    }

    void run_host(const void* src, std::size_t spitch, ObjectId output, void* dst, std::size_t dpitch, int piece) {
        if (prog->units.size() != 1)
            throw Error(ErrorCode::UnsupportedKind, "BandedSession::run_host needs a single-group program");
        const dev::Unit& u = prog->units[0];
        if (unit_ins[0].size() != 1)
            throw Error(ErrorCode::UnsupportedKind, "BandedSession::run_host needs a single-input program");
        const Slab& in = slabs.at(unit_ins[0][0].first);
        const Slab& out = slabs.at(output);
        const int R = unit_ins[0][0].second;
        piece = std::max(piece, 1);
        std::vector<std::pair<int, int>> pieces;
        for (int a = band.row0; a < band.row1; a += piece) pieces.emplace_back(a, std::min(band.row1, a + piece));
        ensure_pipeline(pieces.size());
        const std::size_t in_row = static_cast<std::size_t>(W) * in.bpp, out_row = static_cast<std::size_t>(W) * out.bpp;
        int uploaded = in.row0; // source rows [in.row0, uploaded) are on the device
        const int in_end = in.row0 + in.rows;
        for (std::size_t k = 0; k < pieces.size(); ++k) {
            const auto [a0, a1] = pieces[k];
            const int hi = std::min(in_end, a1 + R);
            if (hi > uploaded) {
                check(gvxb_upload_2d(up, static_cast<char*>(in.ptr) + static_cast<std::int64_t>(uploaded - in.row0) * in.pitch,
                                     static_cast<std::size_t>(in.pitch),
                                     static_cast<const char*>(src) + static_cast<std::size_t>(uploaded - in.row0) * spitch,
                                     spitch, in_row, static_cast<std::size_t>(hi - uploaded)),
                      "band piece upload");
                uploaded = hi;
            }
            check(gvxb_event_record(up, ev_up[k]), "event");
            check(gvxb_stream_wait_event(ctx, ev_up[k]), "event wait");
            compute(u, a0, a1, ctx);
            check(gvxb_event_record(ctx, ev_k[k]), "event");
            check(gvxb_stream_wait_event(dn, ev_k[k]), "event wait");
            check(gvxb_download_2d(dn, static_cast<char*>(dst) + static_cast<std::size_t>(a0 - band.row0) * dpitch, dpitch,
                                   static_cast<const char*>(out.ptr) + static_cast<std::int64_t>(a0 - out.row0) * out.pitch,
                                   static_cast<std::size_t>(out.pitch), out_row, static_cast<std::size_t>(a1 - a0)),
                  "band piece download");
        }
        check(gvxb_sync(dn), "band download sync");
        check(gvxb_sync(ctx), "band compute sync");
    }

    // staging rings of run_host_rows (page-locked, one slot per piece in flight)
    static constexpr int kSlots = 3;
    std::vector<void*> stage_in, stage_out; ///< kSlots each (stage_out: kSlots per output)
    std::size_t stage_in_bytes = 0, stage_out_bytes = 0;
    std::vector<void*> ev_in_free, ev_dn;

    void* staging(std::vector<void*>& ring, std::size_t& have, std::size_t idx, std::size_t bytes, std::size_t count) {
        if (have < bytes || ring.size() < count) {
            check(gvxb_sync(up), "staging sync");
            check(gvxb_sync(dn), "staging sync");
            for (void* q : ring) gvxb_host_free(q);
            ring.assign(count, nullptr);
            for (void*& q : ring) check(gvxb_host_alloc(bytes, &q), "pinned staging allocation");
            have = bytes;
        }
        return ring[idx];
    }

    /// run_host for host rows that may be pageable: input rows are copied
    /// into a page-locked slot (or DMA'd directly when page-locked), output
    /// rows come back through page-locked slots (or directly), each piece's
    /// host copies overlapping the DMA and kernel of its neighbours.  `drain`
    /// (optional, per output) is a second destination filled from a
    /// page-locked `dst` piece by piece.  Returns the device read counter.
    long long run_host_rows(const BandedSession::HostRows& in_rows, const std::vector<BandedSession::HostRows>& outs,
                            int piece) {
        if (prog->units.size() != 1)
            throw Error(ErrorCode::UnsupportedKind, "BandedSession::run_host_rows needs a single-group program");
        const dev::Unit& u = prog->units[0];
        if (unit_ins[0].size() != 1 || unit_ins[0][0].first != in_rows.id)
            throw Error(ErrorCode::UnsupportedKind, "BandedSession::run_host_rows needs the program's single input");
        const Slab& in = slabs.at(in_rows.id);
        const int R = unit_ins[0][0].second;
        piece = std::max(piece, 1);
        std::vector<std::pair<int, int>> pieces;
        for (int a = band.row0; a < band.row1; a += piece) pieces.emplace_back(a, std::min(band.row1, a + piece));
        ensure_pipeline(pieces.size());
        while (ev_dn.size() < pieces.size()) {
            void* e = nullptr;
            check(gvxb_event_create(&e), "event");
            ev_dn.push_back(e);
        }
        while (ev_in_free.size() < static_cast<std::size_t>(kSlots)) {
            void* e = nullptr;
            check(gvxb_event_create(&e), "event");
            ev_in_free.push_back(e);
        }
        std::vector<const Slab*> oslab;
        for (const auto& o : outs) oslab.push_back(&slabs.at(o.id));
        check(gvxb_status_reset(ctx), "status reset");
        const std::size_t in_row = static_cast<std::size_t>(W) * in.bpp;
        const std::size_t max_in = static_cast<std::size_t>(piece + 2 * R) * in_row;
        std::size_t max_out = 0;
        for (const Slab* o : oslab) max_out = std::max(max_out, static_cast<std::size_t>(piece) * W * o->bpp);
        const auto* src = static_cast<const std::uint8_t*>(in_rows.host);
        bool in_used[kSlots] = {false, false, false};
        std::size_t drained = 0; // pieces whose outputs are in their final host place
        auto drain = [&](std::size_t j) {
            const auto [a0, a1] = pieces[j];
            check(gvxb_event_sync(ev_dn[j]), "piece download wait");
            for (std::size_t o = 0; o < outs.size(); ++o) {
                const std::size_t row = static_cast<std::size_t>(W) * oslab[o]->bpp;
                const std::size_t off = static_cast<std::size_t>(a0 - band.row0) * row, n = (a1 - a0) * row;
                auto* dst = static_cast<std::uint8_t*>(outs[o].host);
                if (!outs[o].page_locked) {
                    const void* slot = stage_out[(j % kSlots) * outs.size() + o];
                    dev::parallel_copy(dst + off, slot, n);
                } else if (outs[o].drain) {
                    dev::parallel_copy(static_cast<std::uint8_t*>(outs[o].drain) + off, dst + off, n);
                }
            }
        };
        int uploaded = in.row0;
        const int in_end = in.row0 + in.rows;
        // an error leaves no transfer in flight on the caller's host memory
        struct Quiesce {
            Impl& s;
            bool armed = true;
            ~Quiesce() {
                if (!armed) return;
                gvxb_sync(s.up);
                gvxb_sync(s.dn);
                gvxb_sync(s.ctx);
            }
        } quiesce{*this};
        for (std::size_t k = 0; k < pieces.size(); ++k) {
            const auto [a0, a1] = pieces[k];
            const int hi = std::min(in_end, a1 + R);
            if (hi > uploaded) {
                const std::size_t n = static_cast<std::size_t>(hi - uploaded);
                const std::uint8_t* from = src + static_cast<std::size_t>(uploaded - in.row0) * in_row;
                if (!in_rows.page_locked) {
                    const int slot = static_cast<int>(k % kSlots);
                    void* st = staging(stage_in, stage_in_bytes, slot, max_in, kSlots);
                    if (in_used[slot]) check(gvxb_event_sync(ev_in_free[slot]), "staging wait");
                    dev::parallel_copy(st, from, n * in_row, /*streaming=*/true);
                    from = static_cast<const std::uint8_t*>(st);
                    in_used[slot] = true;
                }
                check(gvxb_upload_2d(up, static_cast<char*>(in.ptr) + static_cast<std::int64_t>(uploaded - in.row0) * in.pitch,
                                     static_cast<std::size_t>(in.pitch), from, in_row, in_row, n),
                      "band piece upload");
                if (!in_rows.page_locked) check(gvxb_event_record(up, ev_in_free[k % kSlots]), "event");
                uploaded = hi;
            }
            check(gvxb_event_record(up, ev_up[k]), "event");
            check(gvxb_stream_wait_event(ctx, ev_up[k]), "event wait");
            compute(u, a0, a1, ctx);
            check(gvxb_event_record(ctx, ev_k[k]), "event");
            check(gvxb_stream_wait_event(dn, ev_k[k]), "event wait");
            // the slot this piece downloads into was last used by piece k - kSlots
            while (drained + kSlots <= k) drain(drained++);
            for (std::size_t o = 0; o < outs.size(); ++o) {
                const Slab& os = *oslab[o];
                const std::size_t row = static_cast<std::size_t>(W) * os.bpp;
                void* to = static_cast<std::uint8_t*>(outs[o].host) + static_cast<std::size_t>(a0 - band.row0) * row;
                if (!outs[o].page_locked) {
                    staging(stage_out, stage_out_bytes, 0, max_out, static_cast<std::size_t>(kSlots) * outs.size());
                    to = stage_out[(k % kSlots) * outs.size() + o];
                }
                check(gvxb_download_2d(dn, to, row,
                                       static_cast<const char*>(os.ptr) + static_cast<std::int64_t>(a0 - os.row0) * os.pitch,
                                       static_cast<std::size_t>(os.pitch), row, static_cast<std::size_t>(a1 - a0)),
                      "band piece download");
            }
            check(gvxb_event_record(dn, ev_dn[k]), "event");
            // host copies of older pieces overlap this piece's transfers
            while (drained + 2 <= k) drain(drained++);
        }
        while (drained < pieces.size()) drain(drained++);
        check(gvxb_sync(up), "band upload sync");
        check(gvxb_sync(ctx), "band compute sync");
        quiesce.armed = false;
        std::uint32_t status = 0;
        long long reads = 0;
        check(gvxb_status_counter_read(ctx, &status, &reads), "device status");
        if (status & GVXB_STATUS_DIV_BY_ZERO) {
            gvxb_status_reset(ctx);
            throw Error(ErrorCode::DivByZero, "division by zero");
        }
        if (status & GVXB_STATUS_INDEX_RANGE) {
            gvxb_status_reset(ctx);
            throw Error(ErrorCode::ShapeMismatch, "array index out of range");
        }
        return reads;
    }

    void synchronize() {
        check(gvxb_sync(ctx), "band sync");
        std::uint32_t status = 0;
        check(gvxb_status_read(ctx, &status), "status read");
        if (status & GVXB_STATUS_DIV_BY_ZERO) {
            gvxb_status_reset(ctx);
            throw Error(ErrorCode::DivByZero, "division by zero in a device kernel");
        }
    }
};

// ------------------------------------------------------------ BandedSession

BandedSession::BandedSession(const OptimizedPlan& plan, int rank, int world, void* comm, int device, int frames)
    : impl_(std::make_unique<Impl>()) {
    impl_->init(plan, rank, world, comm, device, frames);
}

BandedSession::BandedSession() : impl_(std::make_unique<Impl>()) {}

BandedSession::~BandedSession() = default;

namespace detail {

/// run_plan's host path for large frames (execute.cpp): a whole-image band
/// of a program, driven piece by piece from host rows.
struct BandAccess {
    static std::unique_ptr<BandedSession> whole_image(std::shared_ptr<dev::Program> prog) {
        std::unique_ptr<BandedSession> b(new BandedSession());
        b->impl_->init_program(std::move(prog), 0, 1, nullptr, -1, 1);
        const auto& ins = b->impl_->unit_ins;
        if (b->impl_->prog->units.size() != 1 || ins.size() != 1 || ins[0].size() != 1) return nullptr;
        return b;
    }
    static ObjectId input(const BandedSession& b) { return b.impl_->unit_ins[0][0].first; }
    static long long launches(const BandedSession& b) { return gvxb_launch_count(b.impl_->ctx); }
    static int height(const BandedSession& b) { return b.impl_->H; }
};

std::unique_ptr<BandedSession> whole_image_band(std::shared_ptr<dev::Program> prog) {
    try {
        return BandAccess::whole_image(std::move(prog));
    } catch (const Error&) { // not bandable: global operations, run-time scalars, mixed sizes
        return nullptr;
    }
}

ObjectId whole_image_band_input(const BandedSession& b) { return BandAccess::input(b); }
long long whole_image_band_launches(const BandedSession& b) { return BandAccess::launches(b); }

} // namespace detail

BandLayout BandedSession::layout() const {
    BandLayout l;
    l.rank = impl_->rank;
    l.world = impl_->world;
    l.width = impl_->W;
    l.height = impl_->H;
    l.row0 = impl_->band.row0;
    l.row1 = impl_->band.row1;
    const Slab& in = impl_->slabs.at(impl_->input);
    l.src_row0 = in.row0;
    l.src_row1 = in.row0 + in.rows;
    l.halo = impl_->input_halo;
    return l;
}

DeviceTensor BandedSession::tensor(ObjectId id, int* first_row, int* rows) {
    auto it = impl_->slabs.find(id);
    if (it == impl_->slabs.end()) throw Error(ErrorCode::UnknownObject, "object is not an image of the program", id);
    if (first_row) *first_row = it->second.row0;
    if (rows) *rows = it->second.rows;
    return DeviceTensor{it->second.ptr, it->second.pitch, it->second.fstride};
}

void BandedSession::set_stream(void* s) { check(gvxb_ctx_set_stream(impl_->ctx, s), "set stream"); }

void BandedSession::set_overlap(int mode) { check(gvxb_ctx_set_overlap(impl_->ctx, mode), "set overlap"); }

void BandedSession::bind(ObjectId id, DeviceTensor t) {
    auto it = impl_->slabs.find(id);
    if (it == impl_->slabs.end()) throw Error(ErrorCode::UnknownObject, "object is not an image of the program", id);
    Slab& s = it->second;
    const std::int64_t row = static_cast<std::int64_t>(impl_->W) * s.bpp;
    if (!t.data || t.pitch % 16 != 0 || t.pitch < row)
        throw Error(ErrorCode::ShapeMismatch, "band tensor: pitch must be a multiple of 16 and hold a row", id);
    if (impl_->frames > 1 && t.frame_stride < t.pitch * s.rows)
        throw Error(ErrorCode::ShapeMismatch, "band tensor: frame stride too small", id);
    if (s.owned) {
        gvxb_sync(impl_->ctx);
        gvxb_free(impl_->ctx, s.ptr);
    }
    s.ptr = t.data;
    s.pitch = t.pitch;
    s.fstride = impl_->frames > 1 ? t.frame_stride : t.pitch * std::max(1, s.rows);
    s.owned = false;
}

void BandedSession::upload_rows(ObjectId id, const void* host, std::size_t pitch, int first_row, int rows, int frame) {
    auto it = impl_->slabs.find(id);
    if (it == impl_->slabs.end()) throw Error(ErrorCode::UnknownObject, "object is not an image of the program", id);
    const Slab& s = it->second;
    if (first_row < s.row0 || first_row + rows > s.row0 + s.rows || frame < 0 || frame >= impl_->frames)
        throw Error(ErrorCode::ShapeMismatch, "rows outside the band storage", id);
    char* d = static_cast<char*>(s.ptr) + frame * s.fstride + static_cast<std::int64_t>(first_row - s.row0) * s.pitch;
    check(gvxb_upload_2d(impl_->ctx, d, static_cast<std::size_t>(s.pitch), host, pitch,
                         static_cast<std::size_t>(impl_->W) * s.bpp, static_cast<std::size_t>(rows)),
          "band upload");
}

void BandedSession::download_rows(ObjectId id, void* host, std::size_t pitch, int first_row, int rows, int frame) {
    auto it = impl_->slabs.find(id);
    if (it == impl_->slabs.end()) throw Error(ErrorCode::UnknownObject, "object is not an image of the program", id);
    const Slab& s = it->second;
    if (first_row < s.row0 || first_row + rows > s.row0 + s.rows || frame < 0 || frame >= impl_->frames)
        throw Error(ErrorCode::ShapeMismatch, "rows outside the band storage", id);
    const char* d = static_cast<const char*>(s.ptr) + frame * s.fstride +
                    static_cast<std::int64_t>(first_row - s.row0) * s.pitch;
    check(gvxb_download_2d(impl_->ctx, host, pitch, d, static_cast<std::size_t>(s.pitch),
                           static_cast<std::size_t>(impl_->W) * s.bpp, static_cast<std::size_t>(rows)),
          "band download");
    check(gvxb_sync(impl_->ctx), "band download sync");
}

void BandedSession::launch() {
    if (impl_->group) throw Error(ErrorCode::UnsupportedKind, "a BandGroup member launches through its group");
    impl_->launch_standalone();
}

void BandedSession::synchronize() { impl_->synchronize(); }

void BandedSession::run_host(const void* src, std::size_t src_pitch, ObjectId output, void* dst,
                             std::size_t dst_pitch, int piece_rows) {
    impl_->run_host(src, src_pitch, output, dst, dst_pitch, piece_rows);
}

long long BandedSession::run_host_rows(const HostRows& input, const std::vector<HostRows>& outputs, int piece_rows) {
    return impl_->run_host_rows(input, outputs, piece_rows);
}

int BandedSession::launches_per_run() const {
    int n = 0;
    for (std::size_t i = 0; i < impl_->prog->units.size(); ++i) {
        const gvxb_band_plan& p = impl_->unit_plan[i];
        const int per = impl_->prog->units[i].kind == dev::Unit::Kind::Jit
                            ? static_cast<int>(impl_->prog->units[i].prog.kernels.size())
                            : 1;
        n += per * (impl_->has_exchange(i) ? (p.interior_row1 > p.interior_row0 ? 1 : 0) + p.n_edges : 1);
    }
    return n;
}

std::string BandedSession::describe() const {
    std::ostringstream os;
    const BandLayout l = layout();
    os << "row band " << l.rank << "/" << l.world << ": rows [" << l.row0 << ", " << l.row1 << ") of " << l.height
       << ", input slab [" << l.src_row0 << ", " << l.src_row1 << "), halo " << l.halo << "\n"
       << impl_->prog->describe();
    return os.str();
}

// ---------------------------------------------------------------- BandGroup

BandGroup::BandGroup(const OptimizedPlan& plan, const std::vector<int>& devices, int frames) {
    if (devices.empty()) throw Error(ErrorCode::BadKernel, "a band group needs at least one device");
    const int world = static_cast<int>(devices.size());
    auto* ring = new std::vector<BandedSession::Impl*>(); // owned by band 0's Impl lifetime below
    for (int g = 0; g < world; ++g) {
        bands_.push_back(std::make_unique<BandedSession>(plan, g, world, nullptr, devices[static_cast<std::size_t>(g)],
                                                         frames));
        ring->push_back(bands_.back()->impl_.get());
    }
    for (int g = 0; g < world; ++g) {
        BandedSession::Impl& b = *ring->at(static_cast<std::size_t>(g));
        b.group = ring;
        b.index = g;
        b.xctx = dev::own_context(b.device);
        check(gvxb_event_create(&b.ev_ready), "event");
        check(gvxb_event_create(&b.ev_xdone), "event");
        for (int nb : {g - 1, g + 1})
            if (nb >= 0 && nb < world && devices[static_cast<std::size_t>(nb)] != b.device)
                check(gvxb_enable_peer(b.xctx, devices[static_cast<std::size_t>(nb)]), "peer access");
    }
}

BandGroup::~BandGroup() {
    std::vector<BandedSession::Impl*>* ring = bands_.empty() ? nullptr : bands_.front()->impl_->group;
    for (auto& b : bands_) b->impl_->synchronize();
    bands_.clear();
    delete ring;
}

int BandGroup::size() const { return static_cast<int>(bands_.size()); }

BandedSession& BandGroup::band(int g) { return *bands_.at(static_cast<std::size_t>(g)); }

void BandGroup::launch() {
    const std::size_t n_units = bands_.front()->impl_->prog->units.size();
    for (std::size_t i = 0; i < n_units; ++i) {
        bool any = false;
        for (auto& b : bands_) {
            b->impl_->pulled = false;
            if (i == 0) b->impl_->exchanged.clear();
            any = any || b->impl_->needs_exchange(i);
        }
        if (any) {
            for (auto& b : bands_) check(gvxb_event_record(b->impl_->ctx, b->impl_->ev_ready), "exchange event");
            for (auto& b : bands_)
                if (b->impl_->needs_exchange(i)) b->impl_->exchange_peer(i);
        }
        for (auto& b : bands_) b->impl_->run_unit(i, b->impl_->pulled);
        // the next write of this group's inputs (a later group or launch)
        // waits for the neighbours' pulls of them
        for (std::size_t g = 0; g < bands_.size(); ++g)
            for (int nb : {static_cast<int>(g) - 1, static_cast<int>(g) + 1}) {
                if (nb < 0 || nb >= static_cast<int>(bands_.size())) continue;
                BandedSession::Impl* o = bands_[static_cast<std::size_t>(nb)]->impl_.get();
                if (o->pulled) check(gvxb_stream_wait_event(bands_[g]->impl_->ctx, o->ev_xdone), "exchange ordering");
            }
    }
}

void BandGroup::synchronize() {
    for (auto& b : bands_) b->impl_->synchronize();
}

} // namespace gvx
