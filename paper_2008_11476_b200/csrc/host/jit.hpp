// Generic device path: CUDA C emitted from the expression IR of one
// abstraction node and compiled with NVRTC for sm_100a (gvxb_jit_*).
//
// Replaces the reference's per-pixel stack VM (CompiledExpr::run,
// ref:src/expr.cpp:486-519) and the Engine::exec_* loops
// (ref:src/execute.cpp:421-760) for every node that the hand-written fused
// kernels do not cover, and for run_naive.  The emitted code evaluates the
// same tagged int64/double Value semantics (Select stays lazy, casts follow
// cast_value, no FMA contraction: NVRTC runs with --fmad=false), and counts
// pixel-read events exactly like NodeEnv does.
#pragma once

#include "graphvx/kernel.hpp"

#include <cstdint>
#include <string>
#include <vector>

namespace gvx::jit {

/// What a kernel slot is bound to at run time.
enum class SlotKind : std::uint8_t { Image, Scalar, Array, Matrix, None };

struct SlotInfo {
    SlotKind kind = SlotKind::None;
    ResolvedDesc desc;
    bool is_dist = false; ///< array holding a histogram distribution
};

/// One device kernel to launch: NVRTC source + launch geometry.  The single
/// kernel argument is a struct of `nfields` 8-byte fields laid out as the
/// host Binder fills them (see execute.cpp).
struct KernelSpec {
    std::string name;
    std::string source;
    /// Strided: 32-column strips x a few row groups per frame; the kernel
    /// loops over rows and aggregates per block (histograms, reductions).
    enum class Grid : std::uint8_t { Pixels, OutPixels, Single, Rows, Cols, Strided } grid = Grid::Pixels;
    int block_x = 32, block_y = 8;
    int cols = 1; ///< pixels per thread along x (Pixels grids)
    int rows = 1; ///< pixels per thread along y (Pixels grids)
};

/// A node lowered to one or more generated kernels.
struct NodeProgram {
    std::vector<KernelSpec> kernels;
    // field layout of the parameter block:
    //  [0] status*  [1] read counter*  [2] W  [3] H  [4] frame count
    //  then per input slot k: 3 fields (ptr, pitch/len, frame stride)
    //  then per output slot o: 3 fields
    //  then scratch fields (scratch pointer, scratch stride)
    int n_inputs = 0;
    int n_outputs = 0;
    std::size_t scratch_bytes_per_frame = 0; ///< device scratch needed
    bool counts_reads = true;
    int dims_from = -1; ///< input slot giving W/H (-1 = output 0)
    /// Row-band support: rows beyond the output rows each input slot is read
    /// at (window radius, accumulated halo); empty when the program cannot
    /// run on a row band (global reductions, scans, scaling, chains).
    std::vector<int> in_halo;
    //  ... then [fields-4] first output row, [fields-3] end row (row bands;
    //  0 / H for a whole image), [fields-2] scratch pointer, [fields-1] stride
    int fields() const { return 5 + 3 * (n_inputs + n_outputs) + 4; }
};

/// Lowers one abstraction node.  `ins` / `outs` describe the bound objects
/// per INPUT / OUTPUT parameter (None when unbound).  Mask values of a
/// matrix-driven local are taken from `matrix_values` (baked as constants).
/// `count_reads` = false when the host can count the node's reads
/// statically: the kernels then keep no device read counter.
NodeProgram lower_node(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                       const std::vector<SlotInfo>& outs, const std::vector<Value>& matrix_values,
                       bool count_reads = true);

/// One node of a fused region (lower_region).
struct RegionNode {
    const AbstractionKernel* k = nullptr;
    std::vector<SlotInfo> in_slots;  ///< per INPUT parameter
    std::vector<int> in_obj;         ///< per INPUT parameter: region object (shared memory) or -1
    std::vector<int> in_param;       ///< per INPUT parameter: kernel input slot (global) or -1
    std::vector<int> out_obj;        ///< per OUTPUT parameter: region object or -1 (unbound)
    std::vector<Value> matrix;       ///< mask values of a matrix-driven local
};

/// An image produced inside a region: held in shared memory over the tile
/// plus `halo` on each side; `store` >= 0: also written to kernel output
/// slot `store` (consumed outside the region, or observable).
struct RegionObject {
    ImageFormat format = ImageFormat::U8;
    int halo_x = 0, halo_y = 0;
    int store = -1;
    int load = -1; ///< >= 0: an input of the region staged from kernel input slot `load`
    /// a staged input's values are known to lie in [lo, hi] (its producer's
    /// range, e.g. Sobel outputs of a U8 image), narrower than its format's
    bool ranged = false;
    long long lo = 0, hi = 0;
};

/// Whether `e` reads input `slot` through a window (WindowPixel).
bool reads_window(const Expr& e, int slot);

/// A DAG region of point and local nodes over images of one size as ONE
/// kernel (the generic local -> local / point -> local / local -> point
/// fusion): each tile evaluates every node, in topological order, at every
/// position its consumers' windows reach (tile + accumulated halo) into
/// shared memory, each value narrowed to its image's storage format exactly
/// as its store would (SURVEY.md §8a fusion contract rule 1) and taken at
/// the CLAMPED position (rule 2), so every evaluated value is a pixel the
/// reference also computes.  Inputs from outside the region are read from
/// global memory with each reader's border mode.  Nodes are evaluated in
/// their static types (Emitter::temit); throws Error(UnsupportedKind) when a
/// node has run-time-typed parts.  The host counts the events statically.
NodeProgram lower_region(const std::vector<RegionNode>& nodes, const std::vector<RegionObject>& objs,
                         const std::vector<SlotInfo>& ins, const std::vector<SlotInfo>& outs);

} // namespace gvx::jit
