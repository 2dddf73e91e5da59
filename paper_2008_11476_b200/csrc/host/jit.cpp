// CUDA C generator for single abstraction nodes (generic device path).
// See jit.hpp.  Semantics mirrored (file:line in /root/reference/proj):
//   Value arithmetic / casts        src/expr.cpp:8-43, 351-399
//   pixel loads / stores per format src/execute.cpp:36-109
//   window reads, borders, masks    src/execute.cpp:233-254, 550-555
//   point / local / median          src/execute.cpp:421-622
//   reduce (row-major fold, arg)    src/execute.cpp:624-696
//   histogram                       src/execute.cpp:698-727
//   scan / scale / table            src/execute.cpp:729-843
#include "jit.hpp"

#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>

namespace gvx::jit {

namespace {

// ------------------------------------------------------------------ prelude

const char* kPrelude = R"CUDA(
typedef long long i64;
typedef unsigned long long u64;
struct V { int r; i64 i; double f; };
struct P { u64 f[NFIELDS]; };
__device__ __forceinline__ V vi(i64 x) { V v; v.r = 0; v.i = x; v.f = 0.0; return v; }
__device__ __forceinline__ V vf(double x) { V v; v.r = 1; v.i = 0; v.f = x; return v; }
__device__ __forceinline__ double vd(V a) { return a.r ? a.f : __ll2double_rn(a.i); }
__device__ __forceinline__ i64 vl(V a) { return a.r ? (i64)a.f : a.i; }
__device__ __forceinline__ void raise_st(const P& p, unsigned bit) { atomicOr((unsigned*)p.f[0], bit); }
__device__ __forceinline__ V v_add(V a, V b) { return (a.r | b.r) ? vf(__dadd_rn(vd(a), vd(b))) : vi((i64)((u64)a.i + (u64)b.i)); }
__device__ __forceinline__ V v_sub(V a, V b) { return (a.r | b.r) ? vf(__dsub_rn(vd(a), vd(b))) : vi((i64)((u64)a.i - (u64)b.i)); }
__device__ __forceinline__ V v_mul(V a, V b) { return (a.r | b.r) ? vf(__dmul_rn(vd(a), vd(b))) : vi((i64)((u64)a.i * (u64)b.i)); }
__device__ __forceinline__ V v_div(const P& p, V a, V b) {
  if (a.r | b.r) { double d = vd(b); if (d == 0.0) { raise_st(p, 1u); return vf(0.0); } return vf(__ddiv_rn(vd(a), d)); }
  if (b.i == 0) { raise_st(p, 1u); return vi(0); }
  if (b.i == -1) return vi((i64)(0ull - (u64)a.i));
  return vi(a.i / b.i);
}
__device__ __forceinline__ V v_min(V a, V b) {
  if (a.r | b.r) { double x = vd(a), y = vd(b); return vf(y < x ? y : x); }
  return vi(b.i < a.i ? b.i : a.i);
}
__device__ __forceinline__ V v_max(V a, V b) {
  if (a.r | b.r) { double x = vd(a), y = vd(b); return vf(x < y ? y : x); }
  return vi(a.i < b.i ? b.i : a.i);
}
__device__ __forceinline__ i64 shcnt(i64 s) { return s < 0 ? 0 : (s > 63 ? 63 : s); }
__device__ __forceinline__ V v_and(V a, V b) { return vi(a.i & b.i); }
__device__ __forceinline__ V v_or(V a, V b) { return vi(a.i | b.i); }
__device__ __forceinline__ V v_xor(V a, V b) { return vi(a.i ^ b.i); }
__device__ __forceinline__ V v_shl(V a, V b) { return vi((i64)((u64)a.i << shcnt(b.i))); }
__device__ __forceinline__ V v_shr(V a, V b) { return vi(a.i >> shcnt(b.i)); }
__device__ __forceinline__ V v_lt(V a, V b) { return vi((a.r | b.r) ? (vd(a) < vd(b)) : (a.i < b.i)); }
__device__ __forceinline__ V v_gt(V a, V b) { return vi((a.r | b.r) ? (vd(a) > vd(b)) : (a.i > b.i)); }
__device__ __forceinline__ V v_eq(V a, V b) { return vi((a.r | b.r) ? (vd(a) == vd(b)) : (a.i == b.i)); }
__device__ __forceinline__ V v_atan2(V a, V b) { return vf(atan2(vd(a), vd(b))); }
__device__ __forceinline__ V v_not(V a) { return vi(~a.i); }
__device__ __forceinline__ V v_neg(V a) { return a.r ? vf(-a.f) : vi((i64)(0ull - (u64)a.i)); }
__device__ __forceinline__ V v_abs(V a) { return a.r ? vf(fabs(a.f)) : vi(a.i < 0 ? (i64)(0ull - (u64)a.i) : a.i); }
__device__ __forceinline__ V v_sqrt(V a) { return vf(__dsqrt_rn(vd(a))); }
// cast_value: T = 0 U8, 1 U16, 2 S16, 3 S32, 4 F32, 5 I64, 6 F64; pol 0 saturate, 1 wrap
__device__ __forceinline__ V v_cast(V a, int t, int pol) {
  if (t == 6) return vf(vd(a));
  if (t == 4) return vf((double)__double2float_rn(vd(a)));
  if (t == 5) return vi(vl(a));
  i64 lo, hi;
  if (t == 0) { lo = 0; hi = 255; } else if (t == 1) { lo = 0; hi = 65535; }
  else if (t == 2) { lo = -32768; hi = 32767; } else { lo = -2147483648ll; hi = 2147483647ll; }
  i64 x = a.i;
  if (a.r) {
    double r = a.f;
    if (r != r) return vi(0);
    if (pol == 0) {
      if (r >= (double)hi) return vi(hi);
      if (r <= (double)lo) return vi(lo);
      x = llround(r);
    } else {
      x = (i64)fmod(trunc(r), 18446744073709551616.0);
    }
  }
  if (pol == 0) return vi(x < lo ? lo : (x > hi ? hi : x));
  u64 width = (u64)(hi - lo) + 1ull;
  u64 low = (u64)x & (width - 1ull);
  if (lo < 0 && low > (u64)hi) return vi((i64)low - (i64)width);
  return vi((i64)low);
}
__device__ __forceinline__ V ld_val(const i64* slot) {
  // device Value slot: [0] real flag, [1] payload (int64 or double bits)
  return slot[0] ? vf(__longlong_as_double(slot[1])) : vi(slot[1]);
}
__device__ __forceinline__ void st_val(i64* slot, V v) {
  slot[0] = v.r; slot[1] = v.r ? __double_as_longlong(v.f) : v.i;
}
__device__ __forceinline__ void flush_reads(const P& p, u64 rd) {
  for (int o = 16; o > 0; o >>= 1) rd += __shfl_xor_sync(0xffffffffu, rd, o);
  if (((threadIdx.y * blockDim.x + threadIdx.x) & 31) == 0 && rd) atomicAdd((u64*)p.f[1], rd);
}
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
)CUDA";

std::string hex_i64(std::int64_t v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "vi((i64)0x%llxull)", static_cast<unsigned long long>(v));
    return buf;
}

std::string hex_f64(double d) {
    std::uint64_t bits;
    std::memcpy(&bits, &d, 8);
    char buf[64];
    std::snprintf(buf, sizeof buf, "vf(__longlong_as_double((i64)0x%llxull))", static_cast<unsigned long long>(bits));
    return buf;
}

std::string lit(const Value& v) { return v.real ? hex_f64(v.f) : hex_i64(v.i); }

int type_code(ScalarType t) { return static_cast<int>(t); }

int field_in(int k) { return 5 + 3 * k; }

// ------------------------------------------------------------ node emitter

struct Emitter {
    const std::vector<SlotInfo>& ins;
    const std::vector<SlotInfo>& outs;
    int n_in;

    enum class Mode { Point, Tap, Post, Combine, Finalize, BinOf };
    Mode mode = Mode::Point;
    int tdx = 0, tdy = 0;
    const LocalKernel* local = nullptr;
    const std::vector<Value>* mask = nullptr;
    std::ostringstream helpers; // per-slot load functions
    std::vector<std::string> defined;

    Emitter(const std::vector<SlotInfo>& i, const std::vector<SlotInfo>& o)
        : ins(i), outs(o), n_in(static_cast<int>(i.size())) {}

    // Several emitters may share one kernel (fused local chains): this one's
    // input slot s lives at parameter slot `slot_base + s`, its outputs after
    // `n_in_total` inputs, its helpers are named with `prefix`, and reads of
    // input slot `smem_slot` go to `smem_loader` (a shared-memory tile).
    int slot_base = 0;
    int n_in_total = -1;
    std::string prefix;
    int smem_slot = -1;
    std::string smem_loader;
    int fin(int slot) const { return field_in(slot_base + slot); }
    int fout(int o) const { return field_in((n_in_total >= 0 ? n_in_total : n_in) + o); }

    std::string in_base(int slot) const {
        std::ostringstream s;
        s << "((const unsigned char*)p.f[" << fin(slot) << "] + (u64)fr * p.f[" << fin(slot) + 2 << "])";
        return s.str();
    }

    /// Image load function name for (slot, channel, clamp flavour); emitted once.
    std::string image_loader(int slot, Channel ch) {
        if (slot == smem_slot) return smem_loader;
        const SlotInfo& s = ins[static_cast<std::size_t>(slot)];
        std::string name = "ld" + prefix + std::to_string(slot) + "_" + std::to_string(static_cast<int>(ch));
        for (const std::string& d : defined)
            if (d == name) return name;
        defined.push_back(name);
        std::ostringstream f;
        f << "__device__ __forceinline__ V " << name << "(const P& p, int fr, int x, int y, u64& rd) {\n"
          << "  rd++;\n  const unsigned char* row = " << in_base(slot) << " + (u64)y * p.f[" << fin(slot) + 1
          << "];\n";
        switch (s.desc.format) {
        case ImageFormat::U8: f << "  return vi(row[x]);\n"; break;
        case ImageFormat::U16: f << "  return vi(((const unsigned short*)row)[x]);\n"; break;
        case ImageFormat::S16: f << "  return vi(((const short*)row)[x]);\n"; break;
        case ImageFormat::S32: f << "  return vi(((const int*)row)[x]);\n"; break;
        case ImageFormat::F32: f << "  return vf((double)((const float*)row)[x]);\n"; break;
        case ImageFormat::RGB: {
            int c = ch == Channel::G ? 1 : ch == Channel::B ? 2 : 0;
            f << "  return vi(row[3 * x + " << c << "]);\n";
            break;
        }
        case ImageFormat::UYVY:
            if (ch == Channel::U) f << "  return vi(row[4 * (x / 2)]);\n";
            else if (ch == Channel::V) f << "  return vi(row[4 * (x / 2) + 2]);\n";
            else f << "  return vi(row[2 * x + 1]);\n";
            break;
        default: throw Error(ErrorCode::BadFormat, "load from unresolved image");
        }
        f << "}\n";
        helpers << f.str();
        return name;
    }

    std::string scalar_load(int slot) const {
        std::ostringstream s;
        s << "ld_val((const i64*)((const unsigned char*)p.f[" << fin(slot) << "] + (u64)fr * p.f["
          << fin(slot) + 2 << "]))";
        return s.str();
    }

    /// Image slots whose four pixels were loaded into `in<slot>[4]` by a
    /// vector load (point kernels); reads at (px, py) use the registers.
    std::vector<bool> preloaded;

    /// Pointwise read of kernel slot `slot` at (x, y) expressions.
    std::string pointwise(int slot, Channel ch, const std::string& x, const std::string& y) {
        if (slot < 0 || slot >= n_in) throw Error(ErrorCode::TypeMismatch, "input index out of range");
        const SlotInfo& s = ins[static_cast<std::size_t>(slot)];
        if (s.kind == SlotKind::Image && ch == Channel::C0 && x == "px" && y == "py" &&
            static_cast<std::size_t>(slot) < preloaded.size() && preloaded[static_cast<std::size_t>(slot)]) {
            const std::string r = "in" + std::to_string(slot) + "[i]";
            return s.desc.format == ImageFormat::F32 ? "vf((double)" + r + ")" : "vi((i64)" + r + ")";
        }
        switch (s.kind) {
        case SlotKind::Scalar: return scalar_load(slot);
        case SlotKind::Image: return image_loader(slot, ch) + "(p, fr, " + x + ", " + y + ", rd)";
        case SlotKind::None: throw Error(ErrorCode::MissingInput, "read of an unbound input slot");
        default: throw Error(ErrorCode::TypeMismatch, "pointwise read from non-image input");
        }
    }

    std::string array_read(int slot, const std::string& idx) {
        if (slot < 0 || slot >= n_in) throw Error(ErrorCode::TypeMismatch, "array index out of range");
        const SlotInfo& s = ins[static_cast<std::size_t>(slot)];
        if (s.kind != SlotKind::Array && s.kind != SlotKind::Matrix)
            return "(raise_st(p, 2u), vi(0))";
        std::ostringstream o;
        o << "[&]() -> V { i64 at = vl(" << idx << "); u64 n = p.f[" << fin(slot) + 1
          << "]; if (at < 0 || (u64)at >= n) { raise_st(p, 2u); return vi(0); } return ld_val((const i64*)((const "
             "unsigned char*)p.f["
          << fin(slot) << "] + (u64)fr * p.f[" << fin(slot) + 2 << "]) + 2 * at); }()";
        return o.str();
    }

    std::string window(const Expr& e) {
        const int slot = e.input;
        if (slot < 0 || slot >= n_in || ins[static_cast<std::size_t>(slot)].kind != SlotKind::Image)
            throw Error(ErrorCode::TypeMismatch, "window read from non-image input");
        const int ox = tdx + e.dx, oy = tdy + e.dy;
        std::ostringstream x, y;
        x << "(px + (" << ox << "))";
        y << "(py + (" << oy << "))";
        const std::string ld = image_loader(slot, e.channel);
        std::ostringstream o;
        if (local->boundary == BoundaryMode::Constant) {
            o << "([&]() -> V { int xx = " << x.str() << ", yy = " << y.str()
              << "; if (xx < 0 || yy < 0 || xx >= W || yy >= H) return " << lit(local->boundary_value)
              << "; return " << ld << "(p, fr, xx, yy, rd); }())";
        } else {
            o << ld << "(p, fr, clampi(" << x.str() << ", 0, W - 1), clampi(" << y.str() << ", 0, H - 1), rd)";
        }
        return o.str();
    }

    std::string mask_coef(const Expr& e) const {
        const int mw = local->window_w, mh = local->window_h;
        const int ix = std::min(std::max(tdx + e.dx + mw / 2, 0), mw - 1);
        const int iy = std::min(std::max(tdy + e.dy + mh / 2, 0), mh - 1);
        const std::size_t at = static_cast<std::size_t>(iy * mw + ix);
        if (!mask || at >= mask->size()) return "(raise_st(p, 2u), vi(0))";
        return lit((*mask)[at]);
    }

    std::string input(const Expr& e) {
        switch (mode) {
        case Mode::Point:
        case Mode::Tap:
        case Mode::BinOf: return pointwise(e.input, e.channel, "px", "py");
        case Mode::Post: return e.input == 0 ? "cmb" : pointwise(e.input, e.channel, "px", "py");
        case Mode::Combine: return e.input == 0 ? "acc" : "pix";
        case Mode::Finalize:
            if (e.input == 0) return "acc";
            if (e.input == 1) return "vi(cnt)";
            return pointwise(e.input - 1, e.channel, "0", "0");
        }
        return "vi(0)";
    }

    int array_slot(int k) const { return mode == Mode::Finalize ? k - 1 : k; }

    std::string emit(const Expr& e) {
        switch (e.op) {
        case ExprOp::ConstI: return hex_i64(e.ival);
        case ExprOp::ConstF: return hex_f64(e.fval);
        case ExprOp::InputPixel: return input(e);
        case ExprOp::WindowPixel:
            if (mode != Mode::Tap) throw Error(ErrorCode::TypeMismatch, "window read outside a tap body");
            return window(e);
        case ExprOp::MaskCoef:
            if (mode != Mode::Tap) throw Error(ErrorCode::TypeMismatch, "mask read outside a tap body");
            return mask_coef(e);
        case ExprOp::ArrayAt: return array_read(array_slot(e.input), emit(*e.a));
        case ExprOp::Select:
            return "((" + emit(*e.a) + ").i != 0 ? (" + emit(*e.b) + ") : (" + emit(*e.c) + "))";
        case ExprOp::Cast:
            return "v_cast(" + emit(*e.a) + ", " + std::to_string(type_code(e.cast_to)) + ", " +
                   std::to_string(e.policy == CastPolicy::Wrap ? 1 : 0) + ")";
        case ExprOp::Div: return "v_div(p, " + emit(*e.a) + ", " + emit(*e.b) + ")";
        default: break;
        }
        static const char* const bin[] = {"v_add", "v_sub", "v_mul", "",      "v_min", "v_max", "v_and", "v_or",
                                          "v_xor", "v_shl", "v_shr", "v_lt",  "v_gt",  "v_eq",  "v_atan2"};
        if (is_binary(e.op)) {
            const int i = static_cast<int>(e.op) - static_cast<int>(ExprOp::Add);
            return std::string(bin[i]) + "(" + emit(*e.a) + ", " + emit(*e.b) + ")";
        }
        static const char* const un[] = {"v_not", "v_neg", "v_abs", "v_sqrt"};
        const int i = static_cast<int>(e.op) - static_cast<int>(ExprOp::Not);
        return std::string(un[i]) + "(" + emit(*e.a) + ")";
    }

    /// Store statement of V `val` into output slot `o`, channel c (RGB).
    std::string store(int o, const std::string& val, int channel, const std::string& x, const std::string& y) const {
        const SlotInfo& s = outs[static_cast<std::size_t>(o)];
        const int f = fout(o);
        std::ostringstream r;
        r << "{ unsigned char* row = (unsigned char*)p.f[" << f << "] + (u64)fr * p.f[" << f + 2 << "] + (u64)(" << y
          << ") * p.f[" << f + 1 << "]; V sv = " << val << "; ";
        switch (s.desc.format) {
        case ImageFormat::U8: r << "row[" << x << "] = (unsigned char)sv.i;"; break;
        case ImageFormat::U16: r << "((unsigned short*)row)[" << x << "] = (unsigned short)sv.i;"; break;
        case ImageFormat::S16: r << "((short*)row)[" << x << "] = (short)sv.i;"; break;
        case ImageFormat::S32: r << "((int*)row)[" << x << "] = (int)sv.i;"; break;
        case ImageFormat::F32: r << "((float*)row)[" << x << "] = (float)vd(sv);"; break;
        case ImageFormat::RGB: r << "row[3 * (" << x << ") + " << channel << "] = (unsigned char)sv.i;"; break;
        default: throw Error(ErrorCode::BadFormat, "store into unsupported format");
        }
        r << " }\n";
        return r.str();
    }

    std::string out_slot_ptr(int o) const {
        const int f = fout(o);
        return "((i64*)((unsigned char*)p.f[" + std::to_string(f) + "] + (u64)fr * p.f[" + std::to_string(f + 2) +
               "]))";
    }
};

std::string assemble(const Emitter& em, const std::string& body, int nfields) {
    std::string pre = kPrelude;
    const std::string key = "NFIELDS";
    pre.replace(pre.find(key), key.size(), std::to_string(nfields));
    return pre + em.helpers.str() + body;
}

const char* kPixelHead = R"CUDA(
  const int W = (int)p.f[2], H = (int)p.f[3];
  const int px = blockIdx.x * blockDim.x + threadIdx.x;
  const int py = blockIdx.y * blockDim.y + threadIdx.y;
  const int fr = blockIdx.z;
  u64 rd = 0;
  const bool live = px < W && py < H;
)CUDA";

const char* kStridedHead = R"CUDA(
  const int W = (int)p.f[2], H = (int)p.f[3];
  const int px = blockIdx.x * blockDim.x + threadIdx.x;
  const int fr = blockIdx.z;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  u64 rd = 0;
)CUDA";
const char* kStridedLoop =
    "  for (int py = blockIdx.y * blockDim.y + threadIdx.y; py < H; py += gridDim.y * blockDim.y) if (px < W) {\n";

/// Four horizontally adjacent pixels per thread (point / local kernels):
/// address arithmetic, clamps and window loads are shared across them.
constexpr int kCols = 4;
const char* kPixelHead4 = R"CUDA(
  const int W = (int)p.f[2], H = (int)p.f[3];
  const int px4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int py = blockIdx.y * blockDim.y + threadIdx.y;
  const int fr = blockIdx.z;
  u64 rd = 0;
  const bool live = px4 < W && py < H;
)CUDA";
const char* kEachPixel = "#pragma unroll\n    for (int i = 0; i < 4; ++i) { const int px = px4 + i; if (px >= W) break;\n";

// ----------------------------------------------------------------- point

/// Element type and 4-wide vector type of a single-channel image format.
bool vec_types(ImageFormat f, std::string& t, std::string& vt, int& bytes) {
    switch (f) {
    case ImageFormat::U8: t = "unsigned char", vt = "uchar4", bytes = 1; return true;
    case ImageFormat::U16: t = "unsigned short", vt = "ushort4", bytes = 2; return true;
    case ImageFormat::S16: t = "short", vt = "short4", bytes = 2; return true;
    case ImageFormat::S32: t = "int", vt = "int4", bytes = 4; return true;
    case ImageFormat::F32: t = "float", vt = "float4", bytes = 4; return true;
    default: return false;
    }
}

NodeProgram lower_point(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                        const std::vector<SlotInfo>& outs, bool vector_io) {
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    for (std::size_t i = 0; i < ins.size(); ++i)
        if (ins[i].kind == SlotKind::Image) {
            prog.dims_from = static_cast<int>(i);
            break;
        }
    Emitter em(ins, outs);
    em.mode = Emitter::Mode::Point;
    std::ostringstream pre, b, post;
    // vector loads of the four pixels of every single-channel image input
    // (when the host counts the reads; a device read counter needs the
    // per-read loaders), with a scalar fallback at the right edge or for
    // rows that are not vector-aligned
    em.preloaded.assign(ins.size(), false);
    for (std::size_t s = 0; vector_io && s < ins.size(); ++s) {
        std::string t, vt;
        int bytes = 0;
        if (ins[s].kind != SlotKind::Image || !vec_types(ins[s].desc.format, t, vt, bytes)) continue;
        em.preloaded[s] = true;
        pre << "    " << t << " in" << s << "[4];\n    { const " << t << "* r = (const " << t << "*)(" << em.in_base(static_cast<int>(s))
            << " + (u64)py * p.f[" << field_in(static_cast<int>(s)) + 1 << "]) + px4;\n"
            << "      if (px4 + 3 < W && ((u64)r & " << 4 * bytes - 1 << ") == 0) { const " << vt << " v = *(const " << vt
            << "*)r; in" << s << "[0] = v.x; in" << s << "[1] = v.y; in" << s << "[2] = v.z; in" << s << "[3] = v.w; }\n"
            << "      else { for (int i = 0; i < 4; ++i) in" << s << "[i] = px4 + i < W ? r[i] : (" << t << ")0; } }\n";
    }
    const PointKernel& pk = k.point();
    for (std::size_t o = 0; o < pk.outputs.size() && o < outs.size(); ++o) {
        if (outs[o].kind != SlotKind::Image) continue;
        const auto& bodies = pk.outputs[o].channel_bodies;
        std::string t, vt;
        int bytes = 0;
        if (bodies.size() == 3 && outs[o].desc.format == ImageFormat::RGB) {
            for (int c = 0; c < 3; ++c) b << "  " << em.store(static_cast<int>(o), em.emit(*bodies[static_cast<std::size_t>(c)]), c, "px", "py");
        } else if (vector_io && vec_types(outs[o].desc.format, t, vt, bytes)) {
            // the four results gather in registers and leave as one vector store
            const int f = field_in(static_cast<int>(ins.size() + o));
            pre << "    " << t << " out" << o << "[4];\n";
            const std::string cvt = outs[o].desc.format == ImageFormat::F32 ? "(float)vd(sv)" : "(" + t + ")sv.i";
            b << "      { V sv = " << em.emit(*bodies[0]) << "; out" << o << "[i] = " << cvt << "; }\n";
            post << "    { " << t << "* r = (" << t << "*)((unsigned char*)p.f[" << f << "] + (u64)fr * p.f[" << f + 2
                 << "] + (u64)py * p.f[" << f + 1 << "]) + px4;\n"
                 << "      if (px4 + 3 < W && ((u64)r & " << 4 * bytes - 1 << ") == 0) *(" << vt << "*)r = make_" << vt
                 << "(out" << o << "[0], out" << o << "[1], out" << o << "[2], out" << o << "[3]);\n"
                 << "      else { for (int i = 0; i < 4 && px4 + i < W; ++i) r[i] = out" << o << "[i]; } }\n";
        } else {
            b << "  " << em.store(static_cast<int>(o), em.emit(*bodies[0]), 0, "px", "py");
        }
    }
    KernelSpec ks;
    ks.name = "gvx_point";
    ks.cols = kCols;
    std::ostringstream src;
    src << "extern \"C\" __global__ void gvx_point(const P p) {" << kPixelHead4 << "  if (live) {\n" << pre.str()
        << "    " << kEachPixel << b.str() << "    }\n" << post.str() << "  }\n  flush_reads(p, rd);\n}\n";
    ks.source = assemble(em, src.str(), prog.fields());
    prog.kernels.push_back(std::move(ks));
    return prog;
}

// ----------------------------------------------------------------- local

/// Range of an integer image format, or false for non-integer formats.
bool int_format_range(ImageFormat f, std::int64_t& lo, std::int64_t& hi) {
    switch (f) {
    case ImageFormat::U8: lo = 0, hi = 255; return true;
    case ImageFormat::U16: lo = 0, hi = 65535; return true;
    case ImageFormat::S16: lo = -32768, hi = 32767; return true;
    case ImageFormat::S32: lo = -2147483648LL, hi = 2147483647LL; return true;
    default: return false;
    }
}

/// The common shapes of a local tap loop, in exact 32-bit integer
/// arithmetic: Sum of (integer mask coefficient x window pixel) when the
/// worst-case sum fits int32 (then int32 and the reference's int64 agree),
/// or Min / Max of the window pixel.  Clamp borders only.  Emits the body
/// that defines `V cmb` (the combined value) or returns "" when the node
/// does not have such a shape.
std::string int_tap_loop(const LocalKernel& lk, const std::vector<SlotInfo>& ins, const std::vector<Value>& mask,
                         const Emitter& em) {
    if (lk.boundary != BoundaryMode::Clamp || lk.median3x3 || !lk.tap_body) return "";
    const Expr& t = *lk.tap_body;
    const Expr* win = nullptr;
    bool masked = false;
    if (t.op == ExprOp::WindowPixel) {
        win = &t;
    } else if (t.op == ExprOp::Mul && lk.combine == CombineMode::Sum) {
        if (t.a->op == ExprOp::MaskCoef && t.b->op == ExprOp::WindowPixel) win = t.b.get(), masked = true;
        if (t.b->op == ExprOp::MaskCoef && t.a->op == ExprOp::WindowPixel) win = t.a.get(), masked = true;
        const Expr* mc = masked ? (t.a->op == ExprOp::MaskCoef ? t.a.get() : t.b.get()) : nullptr;
        if (mc && (mc->dx != 0 || mc->dy != 0)) return "";
    }
    if (!win || win->channel != Channel::C0 || win->dx != 0 || win->dy != 0) return "";
    const int slot = win->input;
    if (slot < 0 || slot >= static_cast<int>(ins.size()) || ins[static_cast<std::size_t>(slot)].kind != SlotKind::Image)
        return "";
    std::int64_t lo = 0, hi = 0;
    if (!int_format_range(ins[static_cast<std::size_t>(slot)].desc.format, lo, hi)) return "";
    const int ww = lk.window_w, wh = lk.window_h, hw = ww / 2, hh = wh / 2;
    std::vector<std::int64_t> m(static_cast<std::size_t>(ww * wh), 1);
    if (masked) {
        if (mask.size() != m.size()) return "";
        for (std::size_t i = 0; i < m.size(); ++i) {
            if (mask[i].real) return "";
            m[i] = mask[i].i;
            if (m[i] > 2147483647LL || m[i] < -2147483647LL) return "";
        }
    }
    if (lk.combine == CombineMode::Sum) { // every partial sum must fit int32
        std::int64_t bound = 0;
        for (std::int64_t c : m) {
            bound += std::llabs(c) * std::max(std::llabs(lo), std::llabs(hi));
            if (bound > 2147483647LL) return "";
        }
    }
    const char* ctype = "";
    switch (ins[static_cast<std::size_t>(slot)].desc.format) {
    case ImageFormat::U8: ctype = "const unsigned char*"; break;
    case ImageFormat::U16: ctype = "const unsigned short*"; break;
    case ImageFormat::S16: ctype = "const short*"; break;
    default: ctype = "const int*"; break;
    }
    std::ostringstream b;
    // the 4 pixels' windows share 4 + 2 hw clamped columns per window row:
    // every source pixel is loaded once per thread
    const int nc = 4 + 2 * hw;
    for (int k = 0; k < nc; ++k) b << "    const int c" << k << " = clampi(px4 + (" << k - hw << "), 0, W - 1);\n";
    b << "    int acc[4];\n";
    bool first = true;
    const bool sum = lk.combine == CombineMode::Sum;
    for (int dy = -hh; dy <= hh; ++dy) {
        bool used = !sum;
        for (int dx = -hw; dx <= hw && !used; ++dx) used = m[static_cast<std::size_t>((dy + hh) * ww + dx + hw)] != 0;
        if (!used) continue; // an all-zero mask row adds nothing (its reads are still counted)
        b << "    {\n      " << ctype << " r = (" << ctype << ")(" << em.in_base(slot) << " + (u64)clampi(py + (" << dy
          << "), 0, H - 1) * p.f[" << field_in(slot) + 1 << "]);\n      int v[" << nc << "];\n";
        for (int k = 0; k < nc; ++k) b << "      v[" << k << "] = (int)r[c" << k << "];\n";
        b << "#pragma unroll\n      for (int i = 0; i < 4; ++i) {\n";
        for (int dx = -hw; dx <= hw; ++dx) {
            const std::int64_t coef = m[static_cast<std::size_t>((dy + hh) * ww + dx + hw)];
            if (sum && coef == 0) continue;
            std::string term = "v[i + " + std::to_string(dx + hw) + "]";
            if (sum && coef != 1) term = "(" + std::to_string(coef) + " * " + term + ")";
            if (first) b << "        acc[i] = " << term << ";\n";
            else if (sum) b << "        acc[i] += " << term << ";\n";
            else b << "        acc[i] = " << (lk.combine == CombineMode::Min ? "min" : "max") << "(acc[i], " << term << ");\n";
            first = false;
        }
        b << "      }\n    }\n";
    }
    if (first) return ""; // all-zero mask: leave it to the general path
    return b.str();
}

NodeProgram lower_local(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                        const std::vector<SlotInfo>& outs, const std::vector<Value>& matrix_values) {
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    prog.dims_from = -1; // output 0 dims (exec_local iterates the output)
    const LocalKernel& lk = k.local();
    Emitter em(ins, outs);
    em.local = &lk;
    em.mask = lk.mask.empty() ? &matrix_values : &lk.mask;
    const int hw = lk.window_w / 2, hh = lk.window_h / 2;
    const ScalarType out_t = scalar_of(outs.at(0).desc.format);

    std::ostringstream pre, b; // pre: once per thread; b: per pixel (inside the 4-pixel loop)
    if (lk.boundary == BoundaryMode::Undefined) {
        b << "    if (px < " << hw << " || py < " << hh << " || px >= W - " << hw << " || py >= H - " << hh << ") {\n"
          << "      " << em.store(0, "v_cast(vi(0), " + std::to_string(type_code(out_t)) + ", 0)", 0, "px", "py")
          << "      continue;\n    }\n";
    }
    em.mode = Emitter::Mode::Tap;
    const std::string fast = int_tap_loop(lk, ins, *em.mask, em);
    if (!fast.empty()) {
        pre << fast;
        b << "    V cmb = vi((i64)acc[i]);\n";
        prog.counts_reads = false; // the host counts these reads (static window)
    } else if (lk.median3x3) {
        b << "    V t[9];\n";
        int idx = 0;
        for (int dy = -hh; dy <= hh; ++dy)
            for (int dx = -hw; dx <= hw; ++dx) {
                em.tdx = dx;
                em.tdy = dy;
                b << "    t[" << idx++ << "] = " << em.emit(*lk.tap_body) << ";\n";
            }
        b << "    {\n      auto s2 = [](V& a, V& c) { bool sw = (a.r | c.r) ? vd(a) > vd(c) : a.i > c.i; if (sw) { V "
             "tmp = a; a = c; c = tmp; } };\n"
             "      s2(t[1], t[2]); s2(t[4], t[5]); s2(t[7], t[8]); s2(t[0], t[1]); s2(t[3], t[4]); s2(t[6], t[7]);\n"
             "      s2(t[1], t[2]); s2(t[4], t[5]); s2(t[7], t[8]); s2(t[0], t[3]); s2(t[5], t[8]); s2(t[4], t[7]);\n"
             "      s2(t[3], t[6]); s2(t[1], t[4]); s2(t[2], t[5]); s2(t[4], t[7]); s2(t[4], t[2]); s2(t[6], t[4]);\n"
             "      s2(t[4], t[2]);\n    }\n    V cmb = t[4];\n";
    } else {
        const char* comb = lk.combine == CombineMode::Sum ? "v_add" : lk.combine == CombineMode::Min ? "v_min" : "v_max";
        bool first = true;
        for (int dy = -hh; dy <= hh; ++dy)
            for (int dx = -hw; dx <= hw; ++dx) {
                em.tdx = dx;
                em.tdy = dy;
                const std::string v = em.emit(*lk.tap_body);
                if (first) {
                    b << "    V cmb = " << v << ";\n";
                    first = false;
                } else {
                    b << "    cmb = " << comb << "(cmb, " << v << ");\n";
                }
            }
    }
    em.tdx = em.tdy = 0;
    if (lk.post_body) {
        em.mode = Emitter::Mode::Post;
        b << "    " << em.store(0, em.emit(*lk.post_body), 0, "px", "py");
    } else {
        b << "    " << em.store(0, "cmb", 0, "px", "py");
    }
    KernelSpec ks;
    ks.name = "gvx_local";
    ks.cols = kCols;
    std::ostringstream src;
    src << "extern \"C\" __global__ void gvx_local(const P p) {" << kPixelHead4 << "  if (live) {\n" << pre.str()
        << "    " << kEachPixel << b.str() << "    }\n  }\n  flush_reads(p, rd);\n}\n";
    ks.source = assemble(em, src.str(), prog.fields());
    prog.kernels.push_back(std::move(ks));
    return prog;
}

// ------------------------------------------------------- fused local chain

namespace {

/// C type holding a stored pixel of an integer / F32 image format, and the
/// V -> storage conversion of Emitter::store.
bool storage_of(ImageFormat f, std::string& ctype, std::string& conv, std::string& load) {
    switch (f) {
    case ImageFormat::U8: ctype = "unsigned char"; conv = "(unsigned char)sv.i"; load = "vi((i64)v)"; return true;
    case ImageFormat::U16: ctype = "unsigned short"; conv = "(unsigned short)sv.i"; load = "vi((i64)v)"; return true;
    case ImageFormat::S16: ctype = "short"; conv = "(short)sv.i"; load = "vi((i64)v)"; return true;
    case ImageFormat::S32: ctype = "int"; conv = "(int)sv.i"; load = "vi((i64)v)"; return true;
    case ImageFormat::F32: ctype = "float"; conv = "(float)vd(sv)"; load = "vf((double)v)"; return true;
    default: return false;
    }
}

/// Integer fast path of one pixel's tap loop (Clamp border, tap body
/// `window` or `mask * window` with an integer mask whose sums fit int32,
/// integer source format): typed loads and int32 arithmetic, which equal the
/// reference's int64 Value arithmetic there.  A window over the chain's
/// shared-memory intermediate (em.smem_slot) reads the tile (region origin
/// rx0 / ry0, row length rw).  Returns statements defining `V cmb`, or ""
/// when the shape does not apply.
std::string int_tap_single(const LocalKernel& lk, const std::vector<SlotInfo>& ins, const std::vector<Value>& mask,
                           const Emitter& em, int rw) {
    if (lk.boundary != BoundaryMode::Clamp || lk.median3x3 || !lk.tap_body) return "";
    const Expr& t = *lk.tap_body;
    const Expr* win = nullptr;
    bool masked = false;
    if (t.op == ExprOp::WindowPixel) {
        win = &t;
    } else if (t.op == ExprOp::Mul && lk.combine == CombineMode::Sum) {
        if (t.a->op == ExprOp::MaskCoef && t.b->op == ExprOp::WindowPixel) win = t.b.get(), masked = true;
        if (t.b->op == ExprOp::MaskCoef && t.a->op == ExprOp::WindowPixel) win = t.a.get(), masked = true;
        const Expr* mc = masked ? (t.a->op == ExprOp::MaskCoef ? t.a.get() : t.b.get()) : nullptr;
        if (mc && (mc->dx != 0 || mc->dy != 0)) return "";
    }
    if (!win || win->channel != Channel::C0 || win->dx != 0 || win->dy != 0) return "";
    const int slot = win->input;
    if (slot < 0 || slot >= static_cast<int>(ins.size()) || ins[static_cast<std::size_t>(slot)].kind != SlotKind::Image)
        return "";
    std::int64_t lo = 0, hi = 0;
    if (!int_format_range(ins[static_cast<std::size_t>(slot)].desc.format, lo, hi)) return "";
    const int ww = lk.window_w, wh = lk.window_h, hw = ww / 2, hh = wh / 2;
    std::vector<std::int64_t> m(static_cast<std::size_t>(ww * wh), 1);
    if (masked) {
        if (mask.size() != m.size()) return "";
        for (std::size_t i = 0; i < m.size(); ++i) {
            if (mask[i].real) return "";
            m[i] = mask[i].i;
            if (m[i] > 2147483647LL || m[i] < -2147483647LL) return "";
        }
    }
    if (lk.combine == CombineMode::Sum) {
        std::int64_t bound = 0;
        for (std::int64_t c : m) {
            bound += std::llabs(c) * std::max(std::llabs(lo), std::llabs(hi));
            if (bound > 2147483647LL) return "";
        }
    }
    const char* ctype = "";
    switch (ins[static_cast<std::size_t>(slot)].desc.format) {
    case ImageFormat::U8: ctype = "const unsigned char*"; break;
    case ImageFormat::U16: ctype = "const unsigned short*"; break;
    case ImageFormat::S16: ctype = "const short*"; break;
    default: ctype = "const int*"; break;
    }
    const bool smem = slot == em.smem_slot;
    std::ostringstream b;
    b << "    int cacc;\n";
    bool first = true;
    const bool sum = lk.combine == CombineMode::Sum;
    for (int dy = -hh; dy <= hh; ++dy) {
        b << "    {\n";
        if (smem)
            b << "      const int ry = clampi(py + (" << dy << "), 0, H - 1) - ry0;\n";
        else
            b << "      " << ctype << " r = (" << ctype << ")(" << em.in_base(slot) << " + (u64)clampi(py + (" << dy
              << "), 0, H - 1) * p.f[" << em.fin(slot) + 1 << "]);\n";
        for (int dx = -hw; dx <= hw; ++dx) {
            const std::int64_t coef = m[static_cast<std::size_t>((dy + hh) * ww + dx + hw)];
            if (sum && coef == 0) continue;
            std::string v = smem ? "(int)gvx_mid[ry * " + std::to_string(rw) + " + clampi(px + (" + std::to_string(dx) +
                                       "), 0, W - 1) - rx0]"
                                 : "(int)r[clampi(px + (" + std::to_string(dx) + "), 0, W - 1)]";
            if (sum && coef != 1) v = "(" + std::to_string(coef) + " * " + v + ")";
            if (first) b << "      cacc = " << v << ";\n";
            else if (sum) b << "      cacc += " << v << ";\n";
            else b << "      cacc = " << (lk.combine == CombineMode::Min ? "min" : "max") << "(cacc, " << v << ");\n";
            first = false;
        }
        b << "    }\n";
    }
    if (first) return "";
    b << "    V cmb = vi((i64)cacc);\n";
    return b.str();
}

/// Tap loop + post body of a local node at (px, py): statements defining
/// `V pv` (the value before its store).  Integer fast path when it applies,
/// else the Value-typed general path.
std::string local_value(Emitter& em, const LocalKernel& lk, const std::vector<SlotInfo>& ins,
                        const std::vector<Value>& mask, int rw) {
    std::ostringstream b;
    const int hw = lk.window_w / 2, hh = lk.window_h / 2;
    const std::string fast = int_tap_single(lk, ins, mask, em, rw);
    if (!fast.empty()) {
        em.tdx = em.tdy = 0;
        em.mode = Emitter::Mode::Post;
        b << fast << "    V pv = " << (lk.post_body ? em.emit(*lk.post_body) : std::string("cmb")) << ";\n";
        return b.str();
    }
    em.mode = Emitter::Mode::Tap;
    const char* comb = lk.combine == CombineMode::Sum ? "v_add" : lk.combine == CombineMode::Min ? "v_min" : "v_max";
    bool first = true;
    for (int dy = -hh; dy <= hh; ++dy)
        for (int dx = -hw; dx <= hw; ++dx) {
            em.tdx = dx;
            em.tdy = dy;
            const std::string v = em.emit(*lk.tap_body);
            if (first) {
                b << "    V cmb = " << v << ";\n";
                first = false;
            } else {
                b << "    cmb = " << comb << "(cmb, " << v << ");\n";
            }
        }
    em.tdx = em.tdy = 0;
    em.mode = Emitter::Mode::Post;
    b << "    V pv = " << (lk.post_body ? em.emit(*lk.post_body) : std::string("cmb")) << ";\n";
    return b.str();
}

} // namespace
} // namespace (lowering helpers)

bool local_chain_fusible(const AbstractionKernel& producer, const AbstractionKernel& consumer, ImageFormat mid) {
    if (producer.kind != AbstractionKind::Local || consumer.kind != AbstractionKind::Local) return false;
    const LocalKernel& a = producer.local();
    const LocalKernel& b = consumer.local();
    if (a.median3x3 || b.median3x3 || !a.tap_body || !b.tap_body) return false;
    if (a.boundary == BoundaryMode::Undefined || b.boundary != BoundaryMode::Clamp) return false;
    if (b.window_w > 7 || b.window_h > 7 || a.window_w > 7 || a.window_h > 7) return false;
    std::string t, c, l;
    return storage_of(mid, t, c, l);
}

NodeProgram lower_local_chain(const AbstractionKernel& producer, const std::vector<SlotInfo>& p_ins,
                              const std::vector<Value>& p_matrix, const SlotInfo& mid,
                              const AbstractionKernel& consumer, const std::vector<SlotInfo>& c_ins, int c_mid_slot,
                              const std::vector<SlotInfo>& c_outs, const std::vector<Value>& c_matrix) {
    const LocalKernel& pk = producer.local();
    const LocalKernel& ck = consumer.local();
    std::string ctype, conv, load;
    if (!storage_of(mid.desc.format, ctype, conv, load)) throw Error(ErrorCode::BadFormat, "fused chain format");
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(p_ins.size() + c_ins.size());
    prog.n_outputs = static_cast<int>(c_outs.size());
    prog.dims_from = -1;
    prog.counts_reads = false; // static windows: the host counts both nodes' reads
    constexpr int TX = 32, TY = 8;
    const int RX = ck.window_w / 2, RY = ck.window_h / 2;
    const int RW = TX + 2 * RX, RH = TY + 2 * RY;

    std::vector<SlotInfo> p_outs{mid};
    Emitter pe(p_ins, p_outs);
    pe.local = &pk;
    pe.mask = pk.mask.empty() ? &p_matrix : &pk.mask;
    pe.prefix = "P";
    pe.n_in_total = prog.n_inputs;
    Emitter ce(c_ins, c_outs);
    ce.local = &ck;
    ce.mask = ck.mask.empty() ? &c_matrix : &ck.mask;
    ce.prefix = "C";
    ce.slot_base = static_cast<int>(p_ins.size());
    ce.n_in_total = prog.n_inputs;
    ce.smem_slot = c_mid_slot;
    ce.smem_loader = "ld_mid";

    const std::string pbody = local_value(pe, pk, p_ins, *pe.mask, RW);
    const std::string cbody = local_value(ce, ck, c_ins, *ce.mask, RW);
    std::ostringstream src;
    src << "__shared__ " << ctype << " gvx_mid[" << RH * RW << "];\n"
        << "__device__ __forceinline__ V ld_mid(const P& p, int fr, int x, int y, u64& rd) {\n"
        << "  const " << ctype << " v = gvx_mid[(y - ((int)blockIdx.y * " << TY << " - " << RY << ")) * " << RW
        << " + (x - ((int)blockIdx.x * " << TX << " - " << RX << "))];\n  return " << load << ";\n}\n"
        << "extern \"C\" __global__ void gvx_lchain(const P p) {\n"
        << "  const int W = (int)p.f[2], H = (int)p.f[3];\n  const int fr = blockIdx.z;\n  u64 rd = 0;\n"
        << "  const int x0 = (int)blockIdx.x * " << TX << " - " << RX << ", y0 = (int)blockIdx.y * " << TY << " - "
        << RY << ";\n  const int rx0 = x0, ry0 = y0;\n"
        << "  // the intermediate at every (clamped) position the tile's windows read\n"
        << "  for (int e = threadIdx.y * blockDim.x + threadIdx.x; e < " << RH * RW
        << "; e += blockDim.x * blockDim.y) {\n"
        << "    const int px = clampi(x0 + e % " << RW << ", 0, W - 1), py = clampi(y0 + e / " << RW
        << ", 0, H - 1);\n"
        << pbody << "    V sv = pv;\n    gvx_mid[e] = " << conv << ";\n  }\n  __syncthreads();\n"
        << "  const int px = blockIdx.x * " << TX << " + threadIdx.x, py = blockIdx.y * " << TY << " + threadIdx.y;\n"
        << "  if (px < W && py < H) {\n"
        << cbody << "    " << ce.store(0, "pv", 0, "px", "py") << "  }\n}\n";
    KernelSpec ks;
    ks.name = "gvx_lchain";
    ks.block_x = TX;
    ks.block_y = TY;
    ks.cols = 1;
    std::string pre = kPrelude;
    const std::string key = "NFIELDS";
    pre.replace(pre.find(key), key.size(), std::to_string(prog.fields()));
    ks.source = pre + pe.helpers.str() + ce.helpers.str() + src.str();
    prog.kernels.push_back(std::move(ks));
    return prog;
}

namespace {

// ---------------------------------------------------------------- reduce

bool refs_slot(const Expr& e, int slot) {
    if (e.op == ExprOp::InputPixel && e.input == slot) return true;
    for (const ExprPtr* c : {&e.a, &e.b, &e.c})
        if (*c && refs_slot(**c, slot)) return true;
    return false;
}

bool has_real(const Expr& e) {
    if (e.op == ExprOp::ConstF || e.op == ExprOp::Sqrt || e.op == ExprOp::Atan2) return true;
    if (e.op == ExprOp::Cast && (e.cast_to == ScalarType::F32 || e.cast_to == ScalarType::F64)) return true;
    for (const ExprPtr* c : {&e.a, &e.b, &e.c})
        if (*c && has_real(**c)) return true;
    return false;
}

bool has_select_or_div(const Expr& e) {
    if (e.op == ExprOp::Select || e.op == ExprOp::Div || e.op == ExprOp::ArrayAt) return true;
    for (const ExprPtr* c : {&e.a, &e.b, &e.c})
        if (*c && has_select_or_div(**c)) return true;
    return false;
}

NodeProgram lower_reduce(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                         const std::vector<SlotInfo>& outs) {
    const ReduceKernel& rk = k.reduce();
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    prog.dims_from = 0;
    if (ins.empty() || ins[0].kind != SlotKind::Image) throw Error(ErrorCode::TypeMismatch, "reduce needs an image");
    const bool pixel_real = ins[0].desc.format == ImageFormat::F32;
    Emitter em(ins, outs);
    const std::string ldpix = em.image_loader(0, Channel::C0);

    // Parallel forms (exact): integer sum of f(pixel) with init, and
    // seeded min/max (optionally tracking the first arg).
    const Expr& c = *rk.combine;
    bool par_sum = false, par_min = false, par_max = false;
    const Expr* term = nullptr;
    if (!rk.seed_first && !rk.init.real && !pixel_real && c.op == ExprOp::Add && rk.track == ReduceKernel::Track::None) {
        const Expr *l = c.a.get(), *r = c.b.get();
        if (l->op == ExprOp::InputPixel && l->input == 0 && !refs_slot(*r, 0) && !has_real(*r) && !has_select_or_div(*r))
            term = r;
        else if (r->op == ExprOp::InputPixel && r->input == 0 && !refs_slot(*l, 0) && !has_real(*l) &&
                 !has_select_or_div(*l))
            term = l;
        par_sum = term != nullptr;
    }
    if (rk.seed_first && !pixel_real && (c.op == ExprOp::Min || c.op == ExprOp::Max)) {
        const Expr *l = c.a.get(), *r = c.b.get();
        const bool args = l->op == ExprOp::InputPixel && r->op == ExprOp::InputPixel &&
                          ((l->input == 0 && r->input == 1) || (l->input == 1 && r->input == 0));
        if (args) {
            if (c.op == ExprOp::Min && rk.track != ReduceKernel::Track::ArgMax) par_min = true;
            if (c.op == ExprOp::Max && rk.track != ReduceKernel::Track::ArgMin) par_max = true;
        }
    }
    // scratch per frame: [0..1] acc Value, [2] packed key / flag, [3] arg index
    prog.scratch_bytes_per_frame = 64;
    const std::string scratch = "((i64*)((unsigned char*)p.f[" + std::to_string(prog.fields() - 2) +
                                "] + (u64)fr * p.f[" + std::to_string(prog.fields() - 1) + "]))";

    std::ostringstream src;
    // parallel forms: rows strided over a few blocks per frame, per-thread
    // partials, then warp + block aggregation and ONE global atomic per block
    const char* block_sum =
        "  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);\n"
        "  __shared__ i64 red[32];\n  if ((tid & 31) == 0) red[tid >> 5] = part;\n  __syncthreads();\n"
        "  if (tid < 32) { part = tid < (int)((blockDim.x * blockDim.y + 31) >> 5) ? red[tid] : 0;\n"
        "    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o); }\n";
    const char* block_min =
        "  for (int o = 16; o > 0; o >>= 1) { u64 q = __shfl_xor_sync(0xffffffffu, key, o); key = q < key ? q : key; }\n"
        "  __shared__ u64 red[32];\n  if ((tid & 31) == 0) red[tid >> 5] = key;\n  __syncthreads();\n"
        "  if (tid < 32) { key = tid < (int)((blockDim.x * blockDim.y + 31) >> 5) ? red[tid] : ~0ull;\n"
        "    for (int o = 16; o > 0; o >>= 1) { u64 q = __shfl_xor_sync(0xffffffffu, key, o); key = q < key ? q : key; } }\n";
    if (par_sum) {
        em.mode = Emitter::Mode::Combine;
        std::string t = em.emit(*term);
        src << "extern \"C\" __global__ void gvx_reduce_part(const P p) {" << kStridedHead << "  i64 part = 0;\n"
            << kStridedLoop << "    V pix = " << ldpix << "(p, fr, px, py, rd); V acc = vi(0); (void)acc;\n"
            << "    part = (i64)((u64)part + (u64)vl(" << t << "));\n  }\n"
            << block_sum << "  if (tid == 0 && part) atomicAdd((u64*)(" << scratch << " + 1), (u64)part);\n"
            << "  flush_reads(p, rd);\n}\n";
    } else if (par_min || par_max) {
        // key: (biased value, linear index) packed so that atomicMin picks the
        // extreme value and, among equals, the first row-major position
        src << "extern \"C\" __global__ void gvx_reduce_part(const P p) {" << kStridedHead << "  u64 key = ~0ull;\n"
            << kStridedLoop << "    V pix = " << ldpix << "(p, fr, px, py, rd); u64 b = (u64)(pix.i + 2147483648ll);\n"
            << (par_min ? "    u64 kv = b;\n" : "    u64 kv = 0xFFFFFFFFull - b;\n")
            << "    u64 k = (kv << 32) | (u64)(py * (u64)W + px); key = k < key ? k : key;\n  }\n"
            << block_min << "  if (tid == 0 && key != ~0ull) atomicMin((u64*)(" << scratch << " + 2), key);\n"
            << "  flush_reads(p, rd);\n}\n";
    } else {
        // exact row-major fold on one thread (general user combine bodies)
        em.mode = Emitter::Mode::Combine;
        std::string body = em.emit(c);
        const char* cmp = rk.track == ReduceKernel::Track::ArgMin ? "<" : ">";
        src << "extern \"C\" __global__ void gvx_reduce_part(const P p) {\n"
            << "  const int W = (int)p.f[2], H = (int)p.f[3]; const int fr = blockIdx.z; u64 rd = 0;\n"
            << "  if (threadIdx.x != 0 || threadIdx.y != 0) return;\n"
            << "  V acc = " << lit(rk.init) << "; bool seeded = " << (rk.seed_first ? "false" : "true")
            << "; int ax = 0, ay = 0;\n"
            << "  for (int py = 0; py < H; ++py) for (int px = 0; px < W; ++px) {\n"
            << "    V pix = " << ldpix << "(p, fr, px, py, rd);\n"
            << "    if (!seeded) { acc = pix; seeded = true; ax = px; ay = py; continue; }\n";
        if (rk.track != ReduceKernel::Track::None)
            src << "    { bool better = (pix.r | acc.r) ? vd(pix) " << cmp << " vd(acc) : pix.i " << cmp
                << " acc.i; if (better) { ax = px; ay = py; } }\n";
        src << "    acc = " << body << ";\n  }\n"
            << "  st_val(" << scratch << ", acc); " << scratch << "[2] = ax; " << scratch << "[3] = ay;\n"
            << "  atomicAdd((u64*)p.f[1], rd);\n}\n";
    }

    // finalize: one thread per frame
    std::ostringstream fin;
    fin << "extern \"C\" __global__ void gvx_reduce_final(const P p) {\n"
        << "  const int W = (int)p.f[2], H = (int)p.f[3]; const int fr = blockIdx.z; u64 rd = 0; (void)rd;\n"
        << "  if (threadIdx.x != 0) return;\n  const i64 cnt = (i64)W * H;\n  const int px = 0, py = 0; (void)px; (void)py;\n"
        << "  V acc; int ax = 0, ay = 0;\n";
    if (par_sum) {
        fin << "  acc = vi((i64)((u64)" << rk.init.i << "ll + (u64)" << scratch << "[1]));\n";
    } else if (par_min || par_max) {
        fin << "  { u64 key = (u64)" << scratch << "[2]; u64 kv = key >> 32; i64 v = "
            << (par_min ? "(i64)kv" : "(i64)(0xFFFFFFFFull - kv)") << " - 2147483648ll; u64 li = key & 0xFFFFFFFFull;\n"
            << "    if (key == ~0ull) { v = 0; li = 0; }\n"
            << "    acc = vi(v); ax = (int)(li % (u64)W); ay = (int)(li / (u64)W); }\n";
    } else {
        fin << "  acc = ld_val(" << scratch << "); ax = (int)" << scratch << "[2]; ay = (int)" << scratch << "[3];\n";
    }
    if (rk.finalize) {
        em.mode = Emitter::Mode::Finalize;
        fin << "  V res = " << em.emit(*rk.finalize) << ";\n";
    } else {
        fin << "  V res = acc;\n";
    }
    fin << "  if (p.f[" << field_in(prog.n_inputs) << "]) st_val(" << em.out_slot_ptr(0) << ", res);\n";
    if (outs.size() > 1 && rk.track != ReduceKernel::Track::None)
        fin << "  if (p.f[" << field_in(prog.n_inputs + 1) << "]) { i64* l = " << em.out_slot_ptr(1)
            << "; st_val(l, vi(ax)); st_val(l + 2, vi(ay)); }\n";
    fin << "  if (rd) atomicAdd((u64*)p.f[1], rd);\n}\n";

    // init kernel: clear scratch (sum / key) per frame
    std::ostringstream init;
    init << "extern \"C\" __global__ void gvx_reduce_init(const P p) {\n  const int fr = blockIdx.z;\n"
         << "  if (threadIdx.x == 0) { i64* s = " << scratch << "; s[0] = 0; s[1] = 0; s[2] = -1; s[3] = 0; }\n}\n";

    KernelSpec k0, k1, k2;
    k0.name = "gvx_reduce_init";
    k0.grid = KernelSpec::Grid::Single;
    k1.name = "gvx_reduce_part";
    k1.grid = (par_sum || par_min || par_max) ? KernelSpec::Grid::Strided : KernelSpec::Grid::Single;
    k2.name = "gvx_reduce_final";
    k2.grid = KernelSpec::Grid::Single;
    const std::string all = assemble(em, init.str() + src.str() + fin.str(), prog.fields());
    k0.source = all;
    prog.kernels = {k0, k1, k2};
    return prog;
}

// -------------------------------------------------------------- histogram

NodeProgram lower_histogram(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                            const std::vector<SlotInfo>& outs) {
    const HistogramKernel& hk = k.histogram();
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    prog.dims_from = 0;
    Emitter em(ins, outs);
    em.mode = Emitter::Mode::BinOf;
    const std::string bin = em.emit(*hk.bin_of);
    std::ostringstream src;
    src << "extern \"C\" __global__ void gvx_hist_clear(const P p) {\n  const int fr = blockIdx.z;\n"
        << "  i64* o = " << em.out_slot_ptr(0) << ";\n  for (int b = threadIdx.x; b < " << hk.bins
        << "; b += blockDim.x) { o[2 * b] = 0; o[2 * b + 1] = 0; }\n}\n"
        << "extern \"C\" __global__ void gvx_hist(const P p) {";
    const bool smem = hk.bins <= 8192; // per-block u32 counts in shared memory
    if (smem) {
        src << kStridedHead << "  __shared__ unsigned sh[" << hk.bins << "];\n"
            << "  for (int i = tid; i < " << hk.bins << "; i += blockDim.x * blockDim.y) sh[i] = 0;\n  __syncthreads();\n"
            << kStridedLoop << "    i64 b = vl(" << bin << "); if (b >= 0 && b < " << hk.bins << ") atomicAdd(&sh[b], 1u);\n  }\n"
            << "  __syncthreads();\n  i64* o = " << em.out_slot_ptr(0) << ";\n"
            << "  for (int i = tid; i < " << hk.bins << "; i += blockDim.x * blockDim.y) if (sh[i]) atomicAdd((u64*)(o + 2 * i + 1), (u64)sh[i]);\n";
    } else {
        src << kPixelHead << "  if (live) { i64 b = vl(" << bin << "); if (b >= 0 && b < " << hk.bins
            << ") atomicAdd((u64*)(" << em.out_slot_ptr(0) << " + 2 * b + 1), 1ull); }\n";
    }
    src << "  flush_reads(p, rd);\n}\n";
    KernelSpec k0, k1;
    k0.name = "gvx_hist_clear";
    k0.grid = KernelSpec::Grid::Single;
    k0.block_x = 256;
    k1.name = "gvx_hist";
    if (smem) k1.grid = KernelSpec::Grid::Strided;
    k0.source = assemble(em, src.str(), prog.fields());
    prog.kernels = {k0, k1};
    return prog;
}

// ------------------------------------------------------------------ scan

NodeProgram lower_scan(const std::vector<SlotInfo>& ins, const std::vector<SlotInfo>& outs) {
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    prog.dims_from = 0;
    prog.counts_reads = false;
    Emitter em(ins, outs);
    const long long px = static_cast<long long>(ins.at(0).desc.width) * ins.at(0).desc.height;
    const bool parallel = px * 255 <= 2147483647LL; // no S32 saturation possible
    const std::string inb = em.in_base(0);
    const int of = field_in(prog.n_inputs);
    std::ostringstream src;
    src << "__device__ __forceinline__ int* orow(const P& p, int fr, int y) { return (int*)((unsigned char*)p.f[" << of
        << "] + (u64)fr * p.f[" << of + 2 << "] + (u64)y * p.f[" << of + 1 << "]); }\n"
        << "__device__ __forceinline__ int irow(const P& p, int fr, int y, int x) { return (" << inb
        << " + (u64)y * p.f[" << field_in(0) + 1 << "])[x]; }\n";
    if (parallel) {
        src << "extern \"C\" __global__ void gvx_scan_rows(const P p) {\n"
            << "  const int W = (int)p.f[2], H = (int)p.f[3]; const int fr = blockIdx.z;\n"
            << "  const int y = blockIdx.x * blockDim.x + threadIdx.x; if (y >= H) return;\n"
            << "  int s = 0; int* o = orow(p, fr, y); for (int x = 0; x < W; ++x) { s += irow(p, fr, y, x); o[x] = s; }\n}\n"
            << "extern \"C\" __global__ void gvx_scan_cols(const P p) {\n"
            << "  const int W = (int)p.f[2], H = (int)p.f[3]; const int fr = blockIdx.z;\n"
            << "  const int x = blockIdx.x * blockDim.x + threadIdx.x; if (x >= W) return;\n"
            << "  int s = 0; for (int y = 0; y < H; ++y) { int* o = orow(p, fr, y); s += o[x]; o[x] = s; }\n}\n";
        KernelSpec a, b;
        a.name = "gvx_scan_rows";
        a.grid = KernelSpec::Grid::Rows;
        a.block_x = 128;
        a.block_y = 1;
        b.name = "gvx_scan_cols";
        b.grid = KernelSpec::Grid::Cols;
        b.block_x = 128;
        b.block_y = 1;
        a.source = assemble(em, src.str(), prog.fields());
        prog.kernels = {a, b};
    } else {
        // the reference recurrence with S32 saturation at every step
        src << "extern \"C\" __global__ void gvx_scan_seq(const P p) {\n"
            << "  const int W = (int)p.f[2], H = (int)p.f[3]; const int fr = blockIdx.z; if (threadIdx.x) return;\n"
            << "  for (int y = 0; y < H; ++y) for (int x = 0; x < W; ++x) {\n"
            << "    i64 v = irow(p, fr, y, x);\n"
            << "    if (x > 0) v += orow(p, fr, y)[x - 1];\n    if (y > 0) v += orow(p, fr, y - 1)[x];\n"
            << "    if (x > 0 && y > 0) v -= orow(p, fr, y - 1)[x - 1];\n"
            << "    orow(p, fr, y)[x] = (int)(v < -2147483648ll ? -2147483648ll : (v > 2147483647ll ? 2147483647ll : v));\n"
            << "  }\n}\n";
        KernelSpec a;
        a.name = "gvx_scan_seq";
        a.grid = KernelSpec::Grid::Single;
        a.source = assemble(em, src.str(), prog.fields());
        prog.kernels = {a};
    }
    return prog;
}

// ----------------------------------------------------------------- scale

NodeProgram lower_scale(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                        const std::vector<SlotInfo>& outs) {
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    prog.dims_from = -1; // output dims
    prog.counts_reads = false;
    Emitter em(ins, outs);
    const std::string ld = em.image_loader(0, Channel::C0);
    const ResolvedDesc& sd = ins.at(0).desc;
    const ScalarType t = scalar_of(outs.at(0).desc.format);
    std::ostringstream src;
    src << "extern \"C\" __global__ void gvx_scale(const P p) {" << kPixelHead
        << "  const int sw = " << sd.width << ", sh = " << sd.height << ";\n"
        << "  if (live) {\n"
        << "    double yin = __dsub_rn(__ddiv_rn(__dmul_rn((double)py + 0.5, (double)sh), (double)H), 0.5);\n"
        << "    double xin = __dsub_rn(__ddiv_rn(__dmul_rn((double)px + 0.5, (double)sw), (double)W), 0.5);\n"
        << "    V v;\n";
    if (k.scale().interp == InterpMode::Nearest) {
        src << "    int xi = clampi((int)floor(__dadd_rn(xin, 0.5)), 0, sw - 1);\n"
            << "    int yi = clampi((int)floor(__dadd_rn(yin, 0.5)), 0, sh - 1);\n"
            << "    v = " << ld << "(p, fr, xi, yi, rd);\n";
    } else {
        src << "    int x0 = clampi((int)floor(xin), 0, sw - 1), y0 = clampi((int)floor(yin), 0, sh - 1);\n"
            << "    int x1 = min(x0 + 1, sw - 1), y1 = min(y0 + 1, sh - 1);\n"
            << "    double fx = fmin(fmax(__dsub_rn(xin, (double)x0), 0.0), 1.0);\n"
            << "    double fy = fmin(fmax(__dsub_rn(yin, (double)y0), 0.0), 1.0);\n"
            << "    double p00 = vd(" << ld << "(p, fr, x0, y0, rd)), p10 = vd(" << ld << "(p, fr, x1, y0, rd));\n"
            << "    double p01 = vd(" << ld << "(p, fr, x0, y1, rd)), p11 = vd(" << ld << "(p, fr, x1, y1, rd));\n"
            << "    double gx = __dsub_rn(1.0, fx), gy = __dsub_rn(1.0, fy);\n"
            << "    double r = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(p00, gx), gy), "
               "__dmul_rn(__dmul_rn(p10, fx), gy)), __dmul_rn(__dmul_rn(p01, gx), fy)), __dmul_rn(__dmul_rn(p11, fx), fy));\n"
            << "    v = vf(r);\n";
    }
    src << "    " << em.store(0, "v_cast(v, " + std::to_string(type_code(t)) + ", 0)", 0, "px", "py") << "  }\n}\n";
    KernelSpec ks;
    ks.name = "gvx_scale";
    ks.grid = KernelSpec::Grid::OutPixels;
    ks.source = assemble(em, src.str(), prog.fields());
    prog.kernels = {ks};
    return prog;
}

// ----------------------------------------------------------------- table

NodeProgram lower_table(const std::vector<SlotInfo>& ins, const std::vector<SlotInfo>& outs) {
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    prog.counts_reads = false;
    Emitter em(ins, outs);
    std::ostringstream src;
    src << "extern \"C\" __global__ void gvx_table(const P p) {\n  const int fr = blockIdx.z; if (threadIdx.x) return;\n"
        << "  const i64* h = (const i64*)((const unsigned char*)p.f[" << field_in(0) << "] + (u64)fr * p.f[" << field_in(0) + 2
        << "]);\n  const int n = (int)p.f[" << field_in(0) + 1 << "];\n"
        << "  i64* o = " << em.out_slot_ptr(0) << ";\n"
        << "  i64 total = 0; for (int i = 0; i < n; ++i) total += h[2 * i + 1];\n"
        << "  i64 run = 0, cmin = 0; bool found = false;\n"
        << "  for (int i = 0; i < n; ++i) { run += h[2 * i + 1]; if (!found && h[2 * i + 1] > 0) { cmin = run; found = true; } }\n"
        << "  run = 0;\n"
        << "  for (int i = 0; i < n; ++i) {\n    run += h[2 * i + 1]; i64 v;\n"
        << "    if (!found || total == cmin) v = i;\n"
        << "    else v = llround(__ddiv_rn(__dmul_rn(255.0, __ll2double_rn(run - cmin)), __ll2double_rn(total - cmin)));\n"
        << "    v = v < 0 ? 0 : (v > 255 ? 255 : v);\n    st_val(o + 2 * i, vi(v));\n  }\n}\n";
    KernelSpec ks;
    ks.name = "gvx_table";
    ks.grid = KernelSpec::Grid::Single;
    ks.source = assemble(em, src.str(), prog.fields());
    prog.kernels = {ks};
    return prog;
}

} // namespace

NodeProgram lower_node(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                       const std::vector<SlotInfo>& outs, const std::vector<Value>& matrix_values,
                       bool count_reads) {
    NodeProgram p;
    switch (k.kind) {
    case AbstractionKind::Point: p = lower_point(k, ins, outs, /*vector_io=*/!count_reads); break;
    case AbstractionKind::Local: p = lower_local(k, ins, outs, matrix_values); break;
    case AbstractionKind::Reduce: p = lower_reduce(k, ins, outs); break;
    case AbstractionKind::Histogram: p = lower_histogram(k, ins, outs); break;
    case AbstractionKind::Scan: p = lower_scan(ins, outs); break;
    case AbstractionKind::Scale: p = lower_scale(k, ins, outs); break;
    case AbstractionKind::Table: p = lower_table(ins, outs); break;
    }
    if (!count_reads && p.counts_reads) {
        // the host knows the reads statically: drop the per-warp atomic flush
        // of the device read counter (a single-address atomic per warp would
        // otherwise serialise the whole kernel at L2), `rd` then folds away
        const std::string flush = "  flush_reads(p, rd);\n";
        for (KernelSpec& ks : p.kernels)
            for (std::size_t at; (at = ks.source.find(flush)) != std::string::npos;) ks.source.erase(at, flush.size());
        p.counts_reads = false;
    }
    // every kernel of a node shares one source (one NVRTC module)
    for (std::size_t i = 1; i < p.kernels.size(); ++i)
        if (p.kernels[i].source.empty()) p.kernels[i].source = p.kernels[0].source;
    return p;
}

} // namespace gvx::jit
