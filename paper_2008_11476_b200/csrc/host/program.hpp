// Device program: the lowered form of a verified graph (run_naive) or an
// optimized plan (run_plan).  Internal to libgraphvx.
//
// A program is a topologically ordered list of launch units.  A unit is
// either one hand-written fused kernel covering a group of abstraction nodes
// (lower.cpp matches the groups) or one NVRTC-compiled kernel set for one
// node of the executed graph (jit.cpp).  Programs are cached by the verified
// graph's stamp (verify.cpp) plus the values of matrix inputs that are baked
// into generated code.
#pragma once

#include "graphvx/execute.hpp"
#include "graphvx/optimize.hpp"
#include "gvxb.h"
#include "jit.hpp"

#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

namespace gvx::dev {

/// Process-wide device context for the current device (GVX_DEVICE, default
/// 0).  Throws Error(UnsupportedKind) when no CUDA device is present: there
/// is no host execution path.
gvxb_ctx context();

/// Device kernels launched by the process-wide context.
long long launch_count();

/// Throws gvx::Error for a failed C-ABI call.
void check(int status, const char* what);

enum class ArrayRole : std::uint8_t { Plain, Distribution, Location, Table };

struct ObjInfo {
    ObjectId id = kInvalidId;
    ResolvedDesc desc;
    bool is_virtual = false;
    bool produced = false;
    ArrayRole role = ArrayRole::Plain;
    int length = 0;            ///< arrays / matrices: number of Value slots
    int bins = 0;              ///< distributions
    std::int64_t offset = 0, range = 0;
};

struct Unit {
    enum class Kind : std::uint8_t { Jit, Edge, Harris, Stencil, ConvStats } kind = Kind::Jit;
    std::vector<ObjectId> reads, writes;
    std::vector<ObjectId> covers; ///< executed-graph nodes this unit replaces
    std::string label;

    // --- Jit
    AbstractionPtr k;
    std::vector<ObjectId> in_ids, out_ids;
    std::vector<jit::SlotInfo> in_slots, out_slots;
    jit::NodeProgram prog;
    gvxb_module module = nullptr;
    int width = 0, height = 0; ///< working dims of the node

    // --- hand-written kernels
    ObjectId src = kInvalidId;
    ObjectId out[4] = {kInvalidId, kInvalidId, kInvalidId, kInvalidId};
    bool with_gauss = false;
    double k_param = 0.0, threshold = 0.0;
    int ksize = 0;
    int mask[49] = {};
    std::int64_t divisor = 1;
    int mode = 0;
    int conv_format = 2, shift = 0, wrap = 0, bins = 0;
    std::int64_t offset = 0, range = 0;

    // --- reference event counters contributed per frame
    std::int64_t static_reads = 0;
    std::int64_t static_writes = 0;
    bool device_counts_reads = false;
};

struct Program {
    bool naive = false;
    std::vector<Unit> units;
    std::map<ObjectId, ObjInfo> objects; ///< every object a unit touches
    std::string describe() const;
    int launches_per_run(int frames = 1) const;
};

/// Lowers a verified graph to one JIT unit per node (run_naive).
std::shared_ptr<Program> build_naive(const VerifiedGraph& g, const std::map<ObjectId, std::vector<Value>>& matrices);

/// Lowers an optimized plan: hand-written fused groups over the alive
/// implementation nodes, NVRTC units for the remaining fused-graph nodes.
std::shared_ptr<Program> build_plan(const OptimizedPlan& plan,
                                    const std::map<ObjectId, std::vector<Value>>& matrices);

/// The (cached) device program of an optimized plan, as run_plan uses it.
std::shared_ptr<Program> program_of(const OptimizedPlan& plan);

/// A context of its own (stream, status word, read counter) on `device`
/// (-1: the library's device, GVX_DEVICE).
gvxb_ctx own_context(int device = -1);

// ---- hand-written group matching (lower.cpp) --------------------------------

struct GraphView {
    const VerifiedGraph* vg = nullptr;
    const Context* ctx = nullptr;
    std::vector<const OperatorNode*> nodes;         ///< alive nodes, topo order
    std::map<ObjectId, std::vector<ObjectId>> readers; ///< object -> alive nodes reading it
    std::map<ObjectId, ObjectId> writer;               ///< object -> alive producer
    const std::map<ObjectId, std::vector<Value>>* matrices = nullptr;
    bool is_virtual(ObjectId id) const;
    const ResolvedDesc& desc(ObjectId id) const { return vg->desc(id); }
};

/// Hand-written units found in `view`; each unit's `covers` lists base node ids.
std::vector<Unit> match_fused_groups(const GraphView& view);

/// Reference event counts of one executed node (static model), or false when
/// its reads depend on data (image reads under a Select branch).
bool static_counts(const OperatorNode& n, const VerifiedGraph& vg, std::int64_t& reads, std::int64_t& writes);

} // namespace gvx::dev

namespace gvx {
class BandedSession;
}

namespace gvx::detail {

/// Facade-only: the input Buffer `id` is page-locked and still to be filled
/// from `src` (its size); the upload copies and DMAs it chunk by chunk.
struct HostFill {
    ObjectId id = kInvalidId;
    const std::uint8_t* src = nullptr;
    /// optional: image output `drain_id` is also copied into `drain_dst`
    /// during the run (piece by piece); `drained` reports whether it was
    ObjectId drain_id = kInvalidId;
    void* drain_dst = nullptr;
    mutable bool drained = false;
};

/// A BandedSession over the whole image of a single-group, single-input
/// stencil / point program (band.cpp), or null when the program cannot run
/// in row pieces.
std::unique_ptr<BandedSession> whole_image_band(std::shared_ptr<dev::Program> prog);
ObjectId whole_image_band_input(const BandedSession& b);
long long whole_image_band_launches(const BandedSession& b);

/// run_naive / run_plan whose image outputs are downloaded into vectors
/// taken from `out_pool` (keyed by object id, matching size) when present:
/// the C facade keeps page-locked vectors there and hands each report's
/// vectors back before the next run, so outputs DMA straight into them.
ExecutionReport run_naive_pooled(const VerifiedGraph& g, const InputMap& inputs,
                                 std::map<ObjectId, std::vector<std::uint8_t>>* out_pool, const HostFill* fill);
ExecutionReport run_plan_pooled(const OptimizedPlan& plan, const InputMap& inputs,
                                std::map<ObjectId, std::vector<std::uint8_t>>* out_pool, const HostFill* fill);

} // namespace gvx::detail
