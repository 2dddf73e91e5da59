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

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
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
#define ROW0 ((int)p.f[sizeof(p.f) / sizeof(p.f[0]) - 4])
#define ROW1 ((int)p.f[sizeof(p.f) / sizeof(p.f[0]) - 3])
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
// ---- typed forms (Emitter::temit): the same semantics on statically typed
// values, used where a range analysis proves int32 / int64 / double suffice
__device__ __forceinline__ i64 t_cast_d(double r, i64 lo, i64 hi, int pol) {
  if (r != r) return 0;
  if (pol == 0) { if (r >= (double)hi) return hi; if (r <= (double)lo) return lo; return llround(r); }
  i64 x = (i64)fmod(trunc(r), 18446744073709551616.0);
  u64 width = (u64)(hi - lo) + 1ull; u64 low = (u64)x & (width - 1ull);
  return (lo < 0 && low > (u64)hi) ? (i64)low - (i64)width : (i64)low;
}
__device__ __forceinline__ i64 t_sat(i64 x, i64 lo, i64 hi) { return x < lo ? lo : (x > hi ? hi : x); }
// round half away from zero of x / d (d > 0 a literal): llround(x * fl(1/d))
// for |x| < 2^51 when d is odd or a power of two (Emitter::temit, Cast)
__device__ __forceinline__ i64 t_rdiv(i64 x, i64 d) {
  const i64 q = (i64)((2ull * (u64)(x < 0 ? -x : x) + (u64)d) / (2ull * (u64)d)); return x < 0 ? -q : q;
}
__device__ __forceinline__ int t_rdiv32(int x, int d) {
  const int q = (int)((2u * (unsigned)(x < 0 ? -x : x) + (unsigned)d) / (2u * (unsigned)d)); return x < 0 ? -q : q;
}
// llround(sqrt((double)n)) for integer 0 <= n < 2^24: fp32 estimate, then
// the integer correction k* = largest k with k*k - k < n (no n is a half
// square, so half-away rounding never ties)
__device__ __forceinline__ int t_round_sqrt(int n) {
  int k = __float2int_rn(sqrtf(__int2float_rn(n)));
  k -= (k * k - k >= n && k > 0) ? 1 : 0;
  k += (n > k * k + k) ? 1 : 0;
  return k;
}
__device__ __forceinline__ i64 t_wrap(i64 x, i64 lo, i64 hi) {
  u64 width = (u64)(hi - lo) + 1ull; u64 low = (u64)x & (width - 1ull);
  return (lo < 0 && low > (u64)hi) ? (i64)low - (i64)width : (i64)low;
}
__device__ __forceinline__ i64 t_div(const P& p, i64 a, i64 b) {
  if (b == 0) { raise_st(p, 1u); return 0; }
  if (b == -1) return (i64)(0ull - (u64)a);
  return a / b;
}
__device__ __forceinline__ double t_ddiv(const P& p, double a, double d) {
  if (d == 0.0) { raise_st(p, 1u); return 0.0; }
  return __ddiv_rn(a, d);
}
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

/// Static type of a value held in shared memory by a region kernel.
struct TVproto {
    char t = 'i';
    long long lo = 0, hi = 0;
};

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
    /// Region kernels (lower_region): input slot -> parameter slot of the
    /// region kernel, and input slot -> region object held in shared memory
    /// (-1: read from global memory).
    std::vector<int> slot_param;
    std::vector<int> slot_obj;
    /// Shared-memory access of region object o at global (x, y): entry
    /// expression builder set by lower_region.
    std::function<std::string(int, int, int)> obj_entry; ///< (object, dx, dy) from the current entry
    std::function<bool(int, TVproto&)> obj_type;
    int fin(int slot) const {
        return field_in(slot_param.empty() ? slot_base + slot : slot_param[static_cast<std::size_t>(slot)]);
    }
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

    // ------------------------------------------------------------ typed
    // A statically typed form of an expression: 'i' int32, 'l' int64, 'd'
    // double, with the integer value range.  temit() fails (returns false)
    // for anything whose type is only known at run time (scalars / arrays,
    // mixed-type Select, bit ops on reals); callers then use emit().
    struct TV {
        std::string c;
        char t = 'i';
        __int128 lo = 0, hi = 0;
    };
    static constexpr __int128 kI32Lo = -2147483648LL, kI32Hi = 2147483647LL;
    static constexpr __int128 kI64Lo = static_cast<__int128>(INT64_MIN), kI64Hi = static_cast<__int128>(INT64_MAX);
    /// Typed value of the combined tap value in Post mode (slot 0), if any.
    bool cmb_typed = false;
    TV cmb_tv;

    static TV tint(std::string c, __int128 lo, __int128 hi) {
        TV v;
        v.c = std::move(c);
        v.lo = lo;
        v.hi = hi;
        v.t = (lo >= kI32Lo && hi <= kI32Hi) ? 'i' : 'l';
        return v;
    }
    static TV tdbl(std::string c) {
        TV v;
        v.c = std::move(c);
        v.t = 'd';
        return v;
    }
    static std::string as_i64(const TV& v) { return "((i64)(" + v.c + "))"; }
    static std::string as_dbl(const TV& v) { return v.t == 'd' ? v.c : "__ll2double_rn((i64)(" + v.c + "))"; }
    static std::string i128s(__int128 x) {
        // literal of an int64-range bound
        char buf[48];
        std::snprintf(buf, sizeof buf, "((i64)0x%llxull)", static_cast<unsigned long long>(static_cast<long long>(x)));
        return buf;
    }
    static std::string tlit_i(std::int64_t v) {
        char buf[48];
        if (v >= -2147483647LL && v <= 2147483647LL) std::snprintf(buf, sizeof buf, "(%lld)", static_cast<long long>(v));
        else std::snprintf(buf, sizeof buf, "((i64)0x%llxull)", static_cast<unsigned long long>(v));
        return buf;
    }
    static std::string tlit_d(double d) {
        std::uint64_t bits;
        std::memcpy(&bits, &d, 8);
        char buf[64];
        std::snprintf(buf, sizeof buf, "__longlong_as_double((i64)0x%llxull)", static_cast<unsigned long long>(bits));
        return buf;
    }
    static TV tvalue(const Value& v) {
        return v.real ? tdbl(tlit_d(v.f)) : tint(tlit_i(v.i), v.i, v.i);
    }

    /// Typed load of image slot `slot` (int formats -> int, F32 -> double).
    bool typed_loader(int slot, Channel ch, std::string& name, TV& proto) {
        const SlotInfo& s = ins[static_cast<std::size_t>(slot)];
        std::int64_t lo = 0, hi = 255;
        bool real = false;
        const char* expr = nullptr;
        switch (s.desc.format) {
        case ImageFormat::U8: expr = "row[x]"; break;
        case ImageFormat::U16: lo = 0, hi = 65535, expr = "((const unsigned short*)row)[x]"; break;
        case ImageFormat::S16: lo = -32768, hi = 32767, expr = "((const short*)row)[x]"; break;
        case ImageFormat::S32: lo = INT32_MIN, hi = INT32_MAX, expr = "((const int*)row)[x]"; break;
        case ImageFormat::F32: real = true, expr = "(double)((const float*)row)[x]"; break;
        case ImageFormat::RGB:
            expr = ch == Channel::G ? "row[3 * x + 1]" : ch == Channel::B ? "row[3 * x + 2]" : "row[3 * x]";
            break;
        case ImageFormat::UYVY:
            expr = ch == Channel::U ? "row[4 * (x / 2)]" : ch == Channel::V ? "row[4 * (x / 2) + 2]" : "row[2 * x + 1]";
            break;
        default: return false;
        }
        name = "tld" + prefix + std::to_string(slot) + "_" + std::to_string(static_cast<int>(ch));
        proto = real ? tdbl("") : tint("", lo, hi);
        for (const std::string& d : defined)
            if (d == name) return true;
        defined.push_back(name);
        helpers << "__device__ __forceinline__ " << (real ? "double " : "int ") << name
                << "(const P& p, int fr, int x, int y, u64& rd) {\n  rd++;\n  const unsigned char* row = " << in_base(slot)
                << " + (u64)y * p.f[" << fin(slot) + 1 << "];\n  return " << expr << ";\n}\n";
        return true;
    }

    int region_obj(int slot) const {
        return slot_obj.empty() ? -1 : slot_obj[static_cast<std::size_t>(slot)];
    }
    bool tobj(int o, int dx, int dy, TV& out) {
        TVproto pr;
        if (!obj_type || !obj_type(o, pr)) return false;
        const std::string c = obj_entry(o, dx, dy);
        out = pr.t == 'd' ? tdbl("(double)" + c) : tint("(int)" + c, pr.lo, pr.hi);
        return true;
    }

    bool tpointwise(int slot, Channel ch, const std::string& x, const std::string& y, TV& out) {
        if (slot < 0 || slot >= n_in) return false;
        if (region_obj(slot) >= 0) return ch == Channel::C0 && x == "px" && y == "py" && tobj(region_obj(slot), 0, 0, out);
        const SlotInfo& s = ins[static_cast<std::size_t>(slot)];
        if (s.kind != SlotKind::Image || slot == smem_slot) return false;
        if (ch == Channel::C0 && x == "px" && y == "py" && static_cast<std::size_t>(slot) < preloaded.size() &&
            preloaded[static_cast<std::size_t>(slot)]) {
            TV proto;
            std::string name;
            if (!typed_loader(slot, ch, name, proto)) return false;
            const std::string r = "in" + std::to_string(slot) + "[i]";
            out = proto.t == 'd' ? tdbl("(double)" + r) : tint("(int)" + r, proto.lo, proto.hi);
            return true;
        }
        std::string name;
        TV proto;
        if (!typed_loader(slot, ch, name, proto)) return false;
        proto.c = name + "(p, fr, " + x + ", " + y + ", rd)";
        out = proto;
        return true;
    }

    bool twindow(const Expr& e, TV& out) {
        const int slot = e.input;
        if (slot < 0 || slot >= n_in || ins[static_cast<std::size_t>(slot)].kind != SlotKind::Image) return false;
        if (slot == smem_slot) return false;
        const int ox = tdx + e.dx, oy = tdy + e.dy;
        const std::string x = "(px + (" + std::to_string(ox) + "))", y = "(py + (" + std::to_string(oy) + "))";
        if (region_obj(slot) >= 0) {
            // region entries hold the intermediate at the CLAMPED position
            // (Clamp semantics of a virtual intermediate, SURVEY.md §8a rule 2)
            if (e.channel != Channel::C0) return false;
            TV v;
            if (!tobj(region_obj(slot), ox, oy, v)) return false;
            if (local->boundary != BoundaryMode::Constant) {
                out = v;
                return true;
            }
            const Value& bv = local->boundary_value;
            if (bv.real != (v.t == 'd')) return false;
            const std::string ty = v.t == 'd' ? "double" : "i64";
            out = v;
            out.c = "([&]() -> " + ty + " { int xx = " + x + ", yy = " + y +
                    "; if (xx < 0 || yy < 0 || xx >= W || yy >= H) return " + (bv.real ? tlit_d(bv.f) : tlit_i(bv.i)) +
                    "; return " + v.c + "; }())";
            if (!bv.real) {
                out = tint(out.c, std::min<__int128>(v.lo, bv.i), std::max<__int128>(v.hi, bv.i));
                if (out.t == 'i') out.c = "((int)" + out.c + ")";
            }
            return true;
        }
        std::string name;
        TV proto;
        if (!typed_loader(slot, e.channel, name, proto)) return false;
        if (local->boundary == BoundaryMode::Constant) {
            const Value& bv = local->boundary_value;
            if (bv.real != (proto.t == 'd')) return false; // mixed int / real: run-time tags
            const std::string ty = proto.t == 'd' ? "double" : "i64";
            out = proto;
            out.c = "([&]() -> " + ty + " { int xx = " + x + ", yy = " + y +
                    "; if (xx < 0 || yy < 0 || xx >= W || yy >= H) return " +
                    (bv.real ? tlit_d(bv.f) : tlit_i(bv.i)) + "; return " + name + "(p, fr, xx, yy, rd); }())";
            if (!bv.real) {
                out = tint(out.c, std::min<__int128>(proto.lo, bv.i), std::max<__int128>(proto.hi, bv.i));
                if (out.t == 'i') out.c = "((int)" + out.c + ")";
            }
            return true;
        }
        out = proto;
        out.c = name + "(p, fr, clampi(" + x + ", 0, W - 1), clampi(" + y + ", 0, H - 1), rd)";
        return true;
    }

    bool tinput(const Expr& e, TV& out) {
        switch (mode) {
        case Mode::Point:
        case Mode::Tap:
        case Mode::BinOf: return tpointwise(e.input, e.channel, "px", "py", out);
        case Mode::Post:
            if (e.input == 0) {
                if (!cmb_typed) return false;
                out = cmb_tv;
                return true;
            }
            return tpointwise(e.input, e.channel, "px", "py", out);
        default: return false;
        }
    }

    static TV tbin_int(const std::string& op, const TV& a, const TV& b, __int128 lo, __int128 hi) {
        if (lo >= kI64Lo && hi <= kI64Hi) {
            TV r = tint("", lo, hi);
            r.c = r.t == 'i' && a.t == 'i' && b.t == 'i' ? "(" + a.c + " " + op + " " + b.c + ")"
                                                         : "(" + as_i64(a) + " " + op + " " + as_i64(b) + ")";
            return r;
        }
        // may leave int64: the reference's wrapping int64 arithmetic
        TV r = tint("(i64)((u64)" + as_i64(a) + " " + op + " (u64)" + as_i64(b) + ")", kI64Lo, kI64Hi);
        r.t = 'l';
        return r;
    }

    bool temit(const Expr& e, TV& out) {
        switch (e.op) {
        case ExprOp::ConstI: out = tint(tlit_i(e.ival), e.ival, e.ival); return true;
        case ExprOp::ConstF: out = tdbl(tlit_d(e.fval)); return true;
        case ExprOp::InputPixel: return tinput(e, out);
        case ExprOp::WindowPixel: return mode == Mode::Tap && twindow(e, out);
        case ExprOp::MaskCoef: {
            if (mode != Mode::Tap || !mask) return false;
            const int mw = local->window_w, mh = local->window_h;
            const int ix = std::min(std::max(tdx + e.dx + mw / 2, 0), mw - 1);
            const int iy = std::min(std::max(tdy + e.dy + mh / 2, 0), mh - 1);
            const std::size_t at = static_cast<std::size_t>(iy * mw + ix);
            if (at >= mask->size()) return false;
            out = tvalue((*mask)[at]);
            return true;
        }
        case ExprOp::ArrayAt: return false;
        case ExprOp::Select: {
            TV c, x, y;
            if (!temit(*e.a, c) || c.t == 'd' || !temit(*e.b, x) || !temit(*e.c, y)) return false;
            if ((x.t == 'd') != (y.t == 'd')) return false; // the result's tag depends on the branch
            if (x.t == 'd') {
                out = tdbl("((" + c.c + ") != 0 ? " + x.c + " : " + y.c + ")");
                return true;
            }
            out = tint("", std::min(x.lo, y.lo), std::max(x.hi, y.hi));
            out.c = out.t == 'i' ? "((" + c.c + ") != 0 ? " + x.c + " : " + y.c + ")"
                                 : "((" + c.c + ") != 0 ? " + as_i64(x) + " : " + as_i64(y) + ")";
            return true;
        }
        case ExprOp::Cast: {
            TV a;
            if (!temit(*e.a, a)) return false;
            const ScalarType to = e.cast_to;
            if (to == ScalarType::F64) {
                out = tdbl(as_dbl(a));
                return true;
            }
            if (to == ScalarType::F32) {
                if (a.t != 'd' && a.lo >= -16777216 && a.hi <= 16777216) out = tdbl(as_dbl(a)); // exact in float
                else out = tdbl("(double)__double2float_rn(" + as_dbl(a) + ")");
                return true;
            }
            if (to == ScalarType::I64) {
                if (a.t == 'd') out = tint("((i64)(" + a.c + "))", kI64Lo, kI64Hi), out.t = 'l';
                else out = a;
                return true;
            }
            std::int64_t lo = 0, hi = 0;
            switch (to) {
            case ScalarType::U8: lo = 0, hi = 255; break;
            case ScalarType::U16: lo = 0, hi = 65535; break;
            case ScalarType::S16: lo = -32768, hi = 32767; break;
            default: lo = INT32_MIN, hi = INT32_MAX; break;
            }
            const int pol = e.policy == CastPolicy::Wrap ? 1 : 0;
            if (pol == 0 && e.a->op == ExprOp::Sqrt) {
                // cast(int, sqrt(n)) for an integer n in [0, 2^24): exact in fp32
                // plus an integer correction (the reference rounds llround(sqrt(double)))
                TV n;
                if (temit(*e.a->a, n) && n.t != 'd' && n.lo >= 0 && n.hi < (1 << 24)) {
                    const long long kmax = static_cast<long long>(std::sqrt(static_cast<double>(n.hi))) + 1;
                    out = tint("(int)t_sat((i64)t_round_sqrt(" + n.c + "), " + tlit_i(lo) + ", " + tlit_i(hi) + ")",
                               std::max<std::int64_t>(lo, 0), std::min<std::int64_t>(hi, kmax));
                    return true;
                }
            }
            if (pol == 0 && e.a->op == ExprOp::Mul) {
                // cast(int, x * c) with c = fl(1/d): llround(x * c) is the exact
                // half-away rounding of x / d when |x| < 2^51 and d is odd or a
                // power of two (the error stays below the 1/(2d) margin; no ties
                // for odd d) -- an integer division instead of double arithmetic
                const Expr* xe = e.a->a.get();
                const Expr* ce = e.a->b.get();
                if (xe && ce && xe->op == ExprOp::ConstF) std::swap(xe, ce);
                TV x;
                if (xe && ce && ce->op == ExprOp::ConstF && ce->fval > 0 && ce->fval <= 1 && temit(*xe, x) &&
                    x.t != 'd') {
                    const double inv = 1.0 / ce->fval;
                    const long long d = std::llround(inv);
                    const bool odd_or_pow2 = d >= 1 && ((d & 1) || (d & (d - 1)) == 0);
                    const __int128 lim = static_cast<__int128>(1) << 51;
                    if (odd_or_pow2 && d <= (1LL << 30) && 1.0 / static_cast<double>(d) == ce->fval && x.lo > -lim &&
                        x.hi < lim) {
                        const bool i32 = 2 * std::max(-x.lo, x.hi) + d < INT32_MAX;
                        const long long qlo = static_cast<long long>(x.lo / d) - 1, qhi = static_cast<long long>(x.hi / d) + 1;
                        const std::string q = i32 ? "t_rdiv32((int)(" + x.c + "), " + std::to_string(d) + ")"
                                                  : "t_rdiv(" + as_i64(x) + ", " + std::to_string(d) + "LL)";
                        if (qlo >= lo && qhi <= hi) {
                            out = tint("", qlo, qhi);
                            out.c = (out.t == 'i' ? "((int)" : "((i64)") + q + ")";
                        } else {
                            out = tint("(int)t_sat(" + q + ", " + tlit_i(lo) + ", " + tlit_i(hi) + ")",
                                       std::max<long long>(lo, qlo), std::min<long long>(hi, qhi));
                        }
                        return true;
                    }
                }
            }
            if (a.t == 'd') {
                out = tint("(int)t_cast_d(" + a.c + ", " + tlit_i(lo) + ", " + tlit_i(hi) + ", " + std::to_string(pol) + ")",
                           lo, hi);
                return true;
            }
            if (a.lo >= lo && a.hi <= hi) { // already in range: the cast is the identity
                out = a;
                return true;
            }
            if (pol == 0) {
                out = tint("(int)t_sat(" + as_i64(a) + ", " + tlit_i(lo) + ", " + tlit_i(hi) + ")", lo, hi);
            } else {
                out = tint("(int)t_wrap(" + as_i64(a) + ", " + tlit_i(lo) + ", " + tlit_i(hi) + ")", lo, hi);
            }
            return true;
        }
        default: break;
        }
        if (is_binary(e.op)) {
            TV a, b;
            if (!temit(*e.a, a) || !temit(*e.b, b)) return false;
            const bool real = a.t == 'd' || b.t == 'd';
            switch (e.op) {
            case ExprOp::Add:
                if (real) { out = tdbl("__dadd_rn(" + as_dbl(a) + ", " + as_dbl(b) + ")"); return true; }
                out = tbin_int("+", a, b, a.lo + b.lo, a.hi + b.hi);
                return true;
            case ExprOp::Sub:
                if (real) { out = tdbl("__dsub_rn(" + as_dbl(a) + ", " + as_dbl(b) + ")"); return true; }
                out = tbin_int("-", a, b, a.lo - b.hi, a.hi - b.lo);
                return true;
            case ExprOp::Mul: {
                if (real) { out = tdbl("__dmul_rn(" + as_dbl(a) + ", " + as_dbl(b) + ")"); return true; }
                const __int128 p[4] = {a.lo * b.lo, a.lo * b.hi, a.hi * b.lo, a.hi * b.hi};
                __int128 lo = std::min({p[0], p[1], p[2], p[3]}), hi = std::max({p[0], p[1], p[2], p[3]});
                if (a.c == b.c && a.t == b.t) lo = (a.lo <= 0 && a.hi >= 0) ? 0 : std::min(p[0], p[3]); // a square
                out = tbin_int("*", a, b, lo, hi);
                return true;
            }
            case ExprOp::Div: {
                if (real) { out = tdbl("t_ddiv(p, " + as_dbl(a) + ", " + as_dbl(b) + ")"); return true; }
                const __int128 m = std::max(a.lo < 0 ? -a.lo : a.lo, a.hi < 0 ? -a.hi : a.hi);
                out = tint("t_div(p, " + as_i64(a) + ", " + as_i64(b) + ")", -m, m);
                if (out.t == 'i') out.c = "(int)" + out.c;
                return true;
            }
            case ExprOp::Min:
            case ExprOp::Max: {
                const bool mn = e.op == ExprOp::Min;
                if (real) {
                    const std::string x = as_dbl(a), y = as_dbl(b);
                    // v_min / v_max: y < x ? y : x  /  x < y ? y : x
                    out = tdbl("([&]() -> double { double x = " + x + ", y = " + y + "; return " +
                               (mn ? "y < x ? y : x" : "x < y ? y : x") + "; }())");
                    return true;
                }
                out = tint("", mn ? std::min(a.lo, b.lo) : std::max(a.lo, b.lo), mn ? std::min(a.hi, b.hi) : std::max(a.hi, b.hi));
                out.c = std::string(mn ? "min" : "max") + "(" + as_i64(a) + ", " + as_i64(b) + ")";
                if (out.t == 'i') out.c = "(int)" + out.c;
                return true;
            }
            case ExprOp::And:
            case ExprOp::Or:
            case ExprOp::Xor: {
                if (real) return false;
                const char* op = e.op == ExprOp::And ? "&" : e.op == ExprOp::Or ? "|" : "^";
                __int128 lo = kI64Lo, hi = kI64Hi;
                if (a.lo >= 0 && b.lo >= 0) {
                    __int128 m = 1;
                    while (m <= std::max(a.hi, b.hi)) m <<= 1;
                    lo = 0, hi = e.op == ExprOp::And ? std::min(a.hi, b.hi) : m - 1;
                }
                out = tint("(" + as_i64(a) + " " + op + " " + as_i64(b) + ")", lo, hi);
                if (out.t == 'i') out.c = "(int)" + out.c;
                return true;
            }
            case ExprOp::Shl:
                if (real) return false;
                out = tint("(i64)((u64)" + as_i64(a) + " << shcnt(" + as_i64(b) + "))", kI64Lo, kI64Hi);
                out.t = 'l';
                return true;
            case ExprOp::Shr:
                if (real) return false;
                out = tint("(" + as_i64(a) + " >> shcnt(" + as_i64(b) + "))", std::min<__int128>(a.lo, 0),
                           std::max<__int128>(a.hi, 0));
                if (out.t == 'i') out.c = "(int)" + out.c;
                return true;
            case ExprOp::Lt:
            case ExprOp::Gt:
            case ExprOp::Eq: {
                const char* op = e.op == ExprOp::Lt ? "<" : e.op == ExprOp::Gt ? ">" : "==";
                out = real ? tint("(int)(" + as_dbl(a) + " " + op + " " + as_dbl(b) + ")", 0, 1)
                           : tint("(int)(" + as_i64(a) + " " + op + " " + as_i64(b) + ")", 0, 1);
                return true;
            }
            case ExprOp::Atan2: out = tdbl("atan2(" + as_dbl(a) + ", " + as_dbl(b) + ")"); return true;
            default: return false;
            }
        }
        TV a;
        if (!temit(*e.a, a)) return false;
        switch (e.op) {
        case ExprOp::Not:
            if (a.t == 'd') return false;
            out = tint("(~" + as_i64(a) + ")", -a.hi - 1, -a.lo - 1);
            if (out.t == 'i') out.c = "(int)" + out.c;
            return true;
        case ExprOp::Neg:
            if (a.t == 'd') { out = tdbl("(-(" + a.c + "))"); return true; }
            if (a.lo <= kI64Lo) out = tint("(i64)(0ull - (u64)" + as_i64(a) + ")", kI64Lo, kI64Hi), out.t = 'l';
            else out = tint("(-" + as_i64(a) + ")", -a.hi, -a.lo);
            if (out.t == 'i') out.c = "(int)" + out.c;
            return true;
        case ExprOp::Abs:
            if (a.t == 'd') { out = tdbl("fabs(" + a.c + ")"); return true; }
            if (a.lo <= kI64Lo) return false;
            out = tint("", a.lo >= 0 ? a.lo : (a.hi <= 0 ? -a.hi : 0), std::max(a.lo < 0 ? -a.lo : a.lo, a.hi < 0 ? -a.hi : a.hi));
            out.c = "([&]() -> i64 { i64 v = " + as_i64(a) + "; return v < 0 ? -v : v; }())";
            if (out.t == 'i') out.c = "(int)" + out.c;
            return true;
        case ExprOp::Sqrt: out = tdbl("__dsqrt_rn(" + as_dbl(a) + ")"); return true;
        default: return false;
        }
    }

    /// V-typed expression of `e`: the typed form boxed when the analysis
    /// succeeds (the boxes fold away in the compiled code), else emit().
    std::string emit_any(const Expr& e) {
        TV t;
        const std::size_t mark = helpers.tellp();
        const std::size_t ndef = defined.size();
        if (temit(e, t)) return t.t == 'd' ? "vf(" + t.c + ")" : "vi((i64)(" + t.c + "))";
        // drop typed loaders this failed attempt registered
        std::string h = helpers.str();
        h.resize(mark);
        helpers.str(h);
        helpers.seekp(0, std::ios_base::end);
        defined.resize(ndef);
        return emit(e);
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
  const int py = ROW0 + blockIdx.y * blockDim.y + threadIdx.y;
  const int fr = blockIdx.z;
  u64 rd = 0;
  const bool live = px < W && py < ROW1;
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
  const int py = ROW0 + blockIdx.y * blockDim.y + threadIdx.y;
  const int fr = blockIdx.z;
  u64 rd = 0;
  const bool live = px4 < W && py < ROW1;
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
            for (int c = 0; c < 3; ++c) b << "  " << em.store(static_cast<int>(o), em.emit_any(*bodies[static_cast<std::size_t>(c)]), c, "px", "py");
        } else if (vector_io && vec_types(outs[o].desc.format, t, vt, bytes)) {
            // the four results gather in registers and leave as one vector store
            const int f = field_in(static_cast<int>(ins.size() + o));
            pre << "    " << t << " out" << o << "[4];\n";
            const std::string cvt = outs[o].desc.format == ImageFormat::F32 ? "(float)vd(sv)" : "(" + t + ")sv.i";
            b << "      { V sv = " << em.emit_any(*bodies[0]) << "; out" << o << "[i] = " << cvt << "; }\n";
            post << "    { " << t << "* r = (" << t << "*)((unsigned char*)p.f[" << f << "] + (u64)fr * p.f[" << f + 2
                 << "] + (u64)py * p.f[" << f + 1 << "]) + px4;\n"
                 << "      if (px4 + 3 < W && ((u64)r & " << 4 * bytes - 1 << ") == 0) *(" << vt << "*)r = make_" << vt
                 << "(out" << o << "[0], out" << o << "[1], out" << o << "[2], out" << o << "[3]);\n"
                 << "      else { for (int i = 0; i < 4 && px4 + i < W; ++i) r[i] = out" << o << "[i]; } }\n";
        } else {
            b << "  " << em.store(static_cast<int>(o), em.emit_any(*bodies[0]), 0, "px", "py");
        }
    }
    prog.in_halo.assign(ins.size(), 0);
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

/// The tap loop with every tap in its static type (Emitter::temit): int32
/// accumulation when every partial sum's range fits, int64 when it may not
/// (exact: the reference's int64 arithmetic, wrapping alike), double for real
/// taps (same operation order, no contraction).  Returns statements defining
/// `V cmb` and records its typed form for the post body, or "" when some tap
/// has a run-time type (mixed int / real taps included).
std::string typed_combine(Emitter& em, const LocalKernel& lk, const std::vector<Emitter::TV>& taps);

std::string typed_taps(Emitter& em, const LocalKernel& lk) {
    if (!lk.tap_body || lk.median3x3) return "";
    const int hw = lk.window_w / 2, hh = lk.window_h / 2;
    std::vector<Emitter::TV> taps;
    for (int dy = -hh; dy <= hh; ++dy)
        for (int dx = -hw; dx <= hw; ++dx) {
            em.tdx = dx;
            em.tdy = dy;
            Emitter::TV t;
            if (!em.temit(*lk.tap_body, t)) return "";
            taps.push_back(t);
        }
    return typed_combine(em, lk, taps);
}

/// Sum / Min / Max of typed tap values in row-major order (see typed_taps).
std::string typed_combine(Emitter& em, const LocalKernel& lk, const std::vector<Emitter::TV>& all_taps) {
    if (all_taps.empty()) return "";
    // integer sums: a tap that is identically 0 (a zero mask coefficient)
    // adds nothing (its reads are counted by the host)
    std::vector<Emitter::TV> taps;
    for (const Emitter::TV& t : all_taps)
        if (!(lk.combine == CombineMode::Sum && t.t != 'd' && t.lo == 0 && t.hi == 0)) taps.push_back(t);
    if (taps.empty()) taps.push_back(Emitter::tint("0", 0, 0));
    const bool real = taps[0].t == 'd';
    for (const Emitter::TV& t : taps)
        if ((t.t == 'd') != real) return "";
    std::ostringstream b;
    Emitter::TV acc;
    if (real) {
        b << "    double cmbt = " << taps[0].c << ";\n";
        for (std::size_t k = 1; k < taps.size(); ++k) {
            if (lk.combine == CombineMode::Sum) b << "    cmbt = __dadd_rn(cmbt, " << taps[k].c << ");\n";
            else b << "    { double y = " << taps[k].c << "; cmbt = " << (lk.combine == CombineMode::Min ? "y < cmbt ? y : cmbt" : "cmbt < y ? y : cmbt") << "; }\n";
        }
        acc = Emitter::tdbl("cmbt");
        b << "    V cmb = vf(cmbt);\n";
    } else {
        __int128 lo = taps[0].lo, hi = taps[0].hi, plo = lo, phi = hi;
        for (std::size_t k = 1; k < taps.size(); ++k) {
            if (lk.combine == CombineMode::Sum) lo += taps[k].lo, hi += taps[k].hi;
            else if (lk.combine == CombineMode::Min) lo = std::min(lo, taps[k].lo), hi = std::min(hi, taps[k].hi);
            else lo = std::max(lo, taps[k].lo), hi = std::max(hi, taps[k].hi);
            plo = std::min(plo, lo), phi = std::max(phi, hi);
        }
        const bool i32 = plo >= Emitter::kI32Lo && phi <= Emitter::kI32Hi;
        const bool wraps = plo < Emitter::kI64Lo || phi > Emitter::kI64Hi;
        const char* ty = i32 ? "int" : "i64";
        auto term = [&](const Emitter::TV& t) { return i32 ? t.c : Emitter::as_i64(t); };
        b << "    " << ty << " cmbt = " << term(taps[0]) << ";\n";
        for (std::size_t k = 1; k < taps.size(); ++k) {
            if (lk.combine == CombineMode::Sum) {
                if (wraps) b << "    cmbt = (i64)((u64)cmbt + (u64)" << term(taps[k]) << ");\n";
                else b << "    cmbt += " << term(taps[k]) << ";\n";
            } else {
                b << "    cmbt = " << (lk.combine == CombineMode::Min ? "min" : "max") << "(cmbt, " << term(taps[k]) << ");\n";
            }
        }
        acc = wraps ? Emitter::tint("cmbt", Emitter::kI64Lo, Emitter::kI64Hi) : Emitter::tint("cmbt", lo, hi);
        if (!i32) acc.t = 'l';
        b << "    V cmb = vi((i64)cmbt);\n";
    }
    em.cmb_typed = true;
    em.cmb_tv = acc;
    return b.str();
}

namespace {
bool uses_op(const Expr& e, ExprOp op) {
    if (e.op == op) return true;
    for (const ExprPtr* c : {&e.a, &e.b, &e.c})
        if (*c && uses_op(**c, op)) return true;
    return false;
}
} // namespace

/// Local node as a shared-memory tile program (when the host counts its
/// reads statically): the tap body factors as `mask(dx, dy) * g` or `g`,
/// with g a function of the tap position alone (window reads, constants; no
/// pointwise reads of the output pixel, no mask).  g is evaluated ONCE per
/// source position of a 128 x 8 output tile plus its halo, in its static
/// type, into shared memory — a point body the reference fuser inlined into
/// the taps (Multiply -> Box3x3) then costs one evaluation per source pixel
/// instead of one per tap — and each output pixel combines the window from
/// there (row-major, the reference's order and types).  Each window read
/// inside g keeps its own border handling, so the tabulated values are
/// exactly what every tap would compute; only positions some output's window
/// uses are evaluated (no extra DivByZero).  Empty program when the node
/// does not qualify.
NodeProgram lower_local_tiled(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                              const std::vector<SlotInfo>& outs, const std::vector<Value>& matrix_values) {
    NodeProgram none;
    const LocalKernel& lk = k.local();
    if (lk.median3x3 || !lk.tap_body || outs.empty() || outs[0].kind != SlotKind::Image) return none;
    const Expr& t = *lk.tap_body;
    const Expr* g = &t;
    const Expr* mc = nullptr;
    if (t.op == ExprOp::Mul && t.a && t.b) {
        if (t.a->op == ExprOp::MaskCoef && !uses_op(*t.b, ExprOp::MaskCoef)) mc = t.a.get(), g = t.b.get();
        else if (t.b->op == ExprOp::MaskCoef && !uses_op(*t.a, ExprOp::MaskCoef)) mc = t.b.get(), g = t.a.get();
    }
    if (mc && (mc->dx != 0 || mc->dy != 0)) return none;
    if (uses_op(*g, ExprOp::MaskCoef) || uses_op(*g, ExprOp::InputPixel) || uses_op(*g, ExprOp::ArrayAt)) return none;
    // a plain window read is cheaper straight from L1 with the per-thread
    // register reuse of int_tap_loop: tabulate only real computations
    if (g->op == ExprOp::WindowPixel || (g->op == ExprOp::Cast && g->a && g->a->op == ExprOp::WindowPixel)) return none;
    const std::vector<Value>& mask = lk.mask.empty() ? matrix_values : lk.mask;
    const int ww = lk.window_w, wh = lk.window_h, hw = ww / 2, hh = wh / 2;
    if (ww > 9 || wh > 9) return none;
    if (mc && mask.size() != static_cast<std::size_t>(ww * wh)) return none;

    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    prog.dims_from = -1;
    prog.counts_reads = false;
    Emitter em(ins, outs);
    em.local = &lk;
    em.mask = &mask;
    em.mode = Emitter::Mode::Tap;
    em.tdx = em.tdy = 0;
    Emitter::TV gv;
    if (!em.temit(*g, gv)) return none;
    const char* gty = gv.t == 'd' ? "double" : gv.t == 'l' ? "i64" : "int";
    constexpr int TX = 32, TY = 8, PX = 4;
    const int RW = TX * PX + 2 * hw, RH = TY + 2 * hh;
    const bool undef = lk.boundary == BoundaryMode::Undefined;

    // the combine over the tile: tap (dx, dy) of output (threadIdx.x + 32 i, threadIdx.y)
    std::vector<Emitter::TV> taps;
    for (int dy = -hh; dy <= hh; ++dy)
        for (int dx = -hw; dx <= hw; ++dx) {
            Emitter::TV gt = gv;
            gt.c = "gs[(threadIdx.y + " + std::to_string(dy + hh) + ") * " + std::to_string(RW) +
                   " + threadIdx.x + 32 * i + " + std::to_string(dx + hw) + "]";
            if (!mc) {
                taps.push_back(gt);
                continue;
            }
            const Value& cv = mask[static_cast<std::size_t>((dy + hh) * ww + dx + hw)];
            const Emitter::TV cf = Emitter::tvalue(cv);
            if (cv.real || gt.t == 'd') {
                taps.push_back(Emitter::tdbl("__dmul_rn(" + Emitter::as_dbl(cf) + ", " + Emitter::as_dbl(gt) + ")"));
            } else {
                const __int128 pr[4] = {cf.lo * gt.lo, cf.lo * gt.hi, cf.hi * gt.lo, cf.hi * gt.hi};
                taps.push_back(Emitter::tbin_int("*", cf, gt, std::min({pr[0], pr[1], pr[2], pr[3]}),
                                                 std::max({pr[0], pr[1], pr[2], pr[3]})));
            }
        }
    // integer Sum: zero coefficients add nothing (exact); real sums keep every term
    std::vector<Emitter::TV> used;
    for (std::size_t q = 0; q < taps.size(); ++q) {
        const bool zero = mc && lk.combine == CombineMode::Sum && taps[q].t != 'd' && taps[q].lo == 0 && taps[q].hi == 0;
        if (!zero) used.push_back(taps[q]);
    }
    if (used.empty()) return none;
    const std::string comb = typed_combine(em, lk, used);
    if (comb.empty()) return none;
    em.tdx = em.tdy = 0;
    em.mode = Emitter::Mode::Post;
    const std::string pv = lk.post_body ? em.emit_any(*lk.post_body) : std::string("cmb");
    const ScalarType out_t = scalar_of(outs.at(0).desc.format);

    std::ostringstream src;
    src << "extern \"C\" __global__ void gvx_ltile(const P p) {\n"
        << "  const int W = (int)p.f[2], H = (int)p.f[3];\n  const int fr = blockIdx.z;\n  u64 rd = 0;\n"
        << "  const int x0 = (int)blockIdx.x * " << TX * PX << ", y0 = ROW0 + (int)blockIdx.y * " << TY << ";\n"
        << "  __shared__ " << gty << " gs[" << RW * RH << "];\n"
        << "  for (int ry = threadIdx.y; ry < " << RH << "; ry += " << TY << ")\n"
        << "  for (int rx = threadIdx.x; rx < " << RW << "; rx += " << TX << ") {\n"
        << "    const int e = ry * " << RW << " + rx;\n"
        << "    const int px = x0 - " << hw << " + rx, py = y0 - " << hh << " + ry;\n";
    if (undef)
        src << "    if (px < 0 || py < 0 || px >= W || py >= H) continue;\n";
    else
        src << "    if (px < -" << hw << " || py < -" << hh << " || px >= W + " << hw << " || py >= H + " << hh << ") continue;\n";
    src << "    gs[e] = (" << gty << ")(" << gv.c << ");\n  }\n  __syncthreads();\n"
        << "  const int py = y0 + (int)threadIdx.y;\n  if (py >= ROW1) return;\n"
        << "#pragma unroll\n  for (int i = 0; i < " << PX << "; ++i) {\n"
        << "    const int px = x0 + (int)threadIdx.x + " << TX << " * i;\n    if (px >= W) break;\n";
    if (undef)
        src << "    if (px < " << hw << " || py < " << hh << " || px >= W - " << hw << " || py >= H - " << hh << ") {\n"
            << "      " << em.store(0, "v_cast(vi(0), " + std::to_string(type_code(out_t)) + ", 0)", 0, "px", "py")
            << "      continue;\n    }\n";
    src << comb << "    " << em.store(0, pv, 0, "px", "py") << "  }\n  (void)rd;\n}\n";
    prog.in_halo.assign(ins.size(), 0);
    for (std::size_t i = 0; i < ins.size(); ++i)
        if (reads_window(*lk.tap_body, static_cast<int>(i))) prog.in_halo[i] = hh;
    KernelSpec ks;
    ks.name = "gvx_ltile";
    ks.grid = KernelSpec::Grid::Pixels;
    ks.block_x = TX;
    ks.block_y = TY;
    ks.cols = PX;
    ks.source = assemble(em, src.str(), prog.fields());
    prog.kernels.push_back(std::move(ks));
    return prog;
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
    const std::string typed = fast.empty() ? typed_taps(em, lk) : std::string();
    if (!fast.empty()) {
        pre << fast;
        b << "    V cmb = vi((i64)acc[i]);\n";
        prog.counts_reads = false; // the host counts these reads (static window)
        em.cmb_typed = true;
        em.cmb_tv = Emitter::tint("acc[i]", -2147483647LL, 2147483647LL);
    } else if (!typed.empty()) {
        b << typed;
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
        b << "    " << em.store(0, em.emit_any(*lk.post_body), 0, "px", "py");
    } else {
        b << "    " << em.store(0, "cmb", 0, "px", "py");
    }
    prog.in_halo.assign(ins.size(), 0);
    for (std::size_t i = 0; i < ins.size(); ++i)
        if (lk.tap_body && reads_window(*lk.tap_body, static_cast<int>(i))) prog.in_halo[i] = hh;
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

} // namespace (lowering helpers)


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

namespace {
const char* storage_ctype(ImageFormat f) {
    switch (f) {
    case ImageFormat::U8: return "unsigned char";
    case ImageFormat::U16: return "unsigned short";
    case ImageFormat::S16: return "short";
    case ImageFormat::S32: return "int";
    case ImageFormat::F32: return "float";
    default: return nullptr;
    }
}
} // namespace

bool reads_window(const Expr& e, int slot) {
    if (e.op == ExprOp::WindowPixel && e.input == slot) return true;
    for (const ExprPtr* c : {&e.a, &e.b, &e.c})
        if (*c && reads_window(**c, slot)) return true;
    return false;
}

namespace {
bool window_offsets_zero(const Expr& e) {
    if (e.op == ExprOp::WindowPixel && (e.dx != 0 || e.dy != 0)) return false;
    for (const ExprPtr* c : {&e.a, &e.b, &e.c})
        if (*c && !window_offsets_zero(**c)) return false;
    return true;
}
/// A local tap body `mask(dx, dy) * g` or `g` whose g is a computation over
/// window reads at the tap position alone (a point body the reference fuser
/// inlined into the taps): g can be tabulated once per position.  Returns g
/// (and the mask factor, or null) or null when the body does not qualify.
const Expr* tabulated_g(const LocalKernel& lk, const Expr** mc_out) {
    *mc_out = nullptr;
    if (lk.median3x3 || !lk.tap_body) return nullptr;
    const Expr& t = *lk.tap_body;
    const Expr* g = &t;
    const Expr* mc = nullptr;
    if (t.op == ExprOp::Mul && t.a && t.b) {
        if (t.a->op == ExprOp::MaskCoef && !uses_op(*t.b, ExprOp::MaskCoef)) mc = t.a.get(), g = t.b.get();
        else if (t.b->op == ExprOp::MaskCoef && !uses_op(*t.a, ExprOp::MaskCoef)) mc = t.b.get(), g = t.a.get();
    }
    if (mc && (mc->dx != 0 || mc->dy != 0)) return nullptr;
    if (uses_op(*g, ExprOp::MaskCoef) || uses_op(*g, ExprOp::InputPixel) || uses_op(*g, ExprOp::ArrayAt)) return nullptr;
    if (g->op == ExprOp::WindowPixel || (g->op == ExprOp::Cast && g->a && g->a->op == ExprOp::WindowPixel)) return nullptr;
    if (!window_offsets_zero(*g)) return nullptr;
    *mc_out = mc;
    return g;
}
} // namespace

namespace {

/// One region kernel at a given tile (TW x TH outputs per 256-thread block);
/// `smem` receives the static shared memory the emitted kernel declares.
NodeProgram lower_region_at(const std::vector<RegionNode>& nodes, const std::vector<RegionObject>& objs,
                            const std::vector<SlotInfo>& ins, const std::vector<SlotInfo>& outs, const int TW,
                            const int TH, std::size_t& smem) {
    auto unsupported = [](const std::string& why) { return Error(ErrorCode::UnsupportedKind, "region: " + why); };
    for (const RegionObject& o : objs)
        if (!storage_ctype(o.format)) throw unsupported("intermediate format");
    // nodes whose tap computation is tabulated per position (see tabulated_g)
    std::vector<bool> tab(nodes.size(), false);
    static const bool tab_on = std::getenv("GVX_REGION_TAB") != nullptr; // measured slower on the corpus
    for (std::size_t ni = 0; ni < nodes.size() && tab_on; ++ni) {
        if (nodes[ni].k->kind != AbstractionKind::Local) continue;
        const Expr* mc = nullptr;
        tab[ni] = tabulated_g(nodes[ni].k->local(), &mc) != nullptr;
    }
    NodeProgram prog;
    prog.n_inputs = static_cast<int>(ins.size());
    prog.n_outputs = static_cast<int>(outs.size());
    prog.dims_from = -1;
    prog.counts_reads = false;
    // staged inputs are laid out from a 16-byte-aligned column origin
    // (colofs >= halo, in elements) so interior tiles copy them with 16-byte
    // vector loads and stores; other objects start at their halo
    static const bool vec_on = std::getenv("GVX_REGION_NOVEC") == nullptr;
    auto colofs = [&](int o) {
        const RegionObject& O = objs[static_cast<std::size_t>(o)];
        const int es = bytes_per_pixel(O.format), per = 16 / std::max(es, 1);
        if (O.load < 0 || !vec_on || es > 16 || 16 % es) return O.halo_x;
        return (O.halo_x + per - 1) / per * per;
    };
    auto rw = [&](int o) { return TW + 2 * colofs(o); };
    auto rh = [&](int o) { return TH + 2 * objs[static_cast<std::size_t>(o)].halo_y; };
    // a node's code reads object o relative to the entry being evaluated:
    // index base b<o> (set per entry) + dy * row length + dx
    std::vector<bool> used_obj(objs.size());
    // point nodes evaluated inside their consumers (see the node loop): the
    // object's value is its producer's expression at the same entry
    std::vector<bool> inline_obj(objs.size(), false);
    std::vector<std::string> inline_code(objs.size());
    std::vector<std::vector<int>> inline_uses(objs.size());
    std::function<std::string(int, int, int)> entry = [&](int o, int dx, int dy) -> std::string {
        if (inline_obj[static_cast<std::size_t>(o)]) {
            for (int u : inline_uses[static_cast<std::size_t>(o)]) used_obj[static_cast<std::size_t>(u)] = true;
            return inline_code[static_cast<std::size_t>(o)];
        }
        used_obj[static_cast<std::size_t>(o)] = true;
        return "ro" + std::to_string(o) + "[b" + std::to_string(o) + " + (" + std::to_string(dy * rw(o) + dx) + ")]";
    };
    // value ranges of the entries: the format's, narrowed to the producing
    // node's static range when it stores without narrowing
    std::vector<TVproto> orange(objs.size());
    for (std::size_t o = 0; o < objs.size(); ++o) {
        std::int64_t lo = 0, hi = 0;
        if (objs[o].format == ImageFormat::F32) orange[o].t = 'd';
        else if (int_format_range(objs[o].format, lo, hi)) orange[o].lo = lo, orange[o].hi = hi;
        if (objs[o].ranged && orange[o].t != 'd' && objs[o].lo >= orange[o].lo && objs[o].hi <= orange[o].hi)
            orange[o].lo = objs[o].lo, orange[o].hi = objs[o].hi;
    }
    auto otype = [&](int o, TVproto& pr) {
        pr = orange[static_cast<std::size_t>(o)];
        return true;
    };

    // point nodes evaluated inside their consumers (pre-pass: their objects
    // get no shared memory): outputs read only at the same entry by later
    // nodes (no halo, not stored), bodies that cannot raise
    static const bool inline_on = std::getenv("GVX_REGION_NOINLINE") == nullptr;
    std::vector<bool> inline_node(nodes.size(), false);
    for (std::size_t ni = 0; ni < nodes.size() && inline_on; ++ni) {
        const RegionNode& rn = nodes[ni];
        if (rn.k->kind != AbstractionKind::Point) continue;
        const PointKernel& pk = rn.k->point();
        bool ok = false;
        for (std::size_t j = 0; j < rn.out_obj.size(); ++j) {
            const int o = rn.out_obj[j];
            if (o < 0) continue;
            const RegionObject& O = objs[static_cast<std::size_t>(o)];
            ok = O.halo_x == 0 && O.halo_y == 0 && O.store < 0 && O.load < 0 && j < pk.outputs.size() &&
                 pk.outputs[j].channel_bodies.size() == 1 && !uses_op(*pk.outputs[j].channel_bodies[0], ExprOp::Div) &&
                 !uses_op(*pk.outputs[j].channel_bodies[0], ExprOp::ArrayAt);
            if (!ok) break;
        }
        if (!ok) continue;
        inline_node[ni] = true;
        for (int o : rn.out_obj)
            if (o >= 0) inline_obj[static_cast<std::size_t>(o)] = true;
    }

    std::ostringstream helpers, body;
    body << "extern \"C\" __global__ void gvx_region(const P p) {\n"
         << "  const int W = (int)p.f[2], H = (int)p.f[3];\n  const int fr = blockIdx.z;\n  u64 rd = 0;\n"
         << "  const int tx0 = (int)blockIdx.x * " << TW << ", ty0 = ROW0 + (int)blockIdx.y * " << TH << ";\n";
    for (std::size_t o = 0; o < objs.size(); ++o)
        if (!inline_obj[o])
            body << "  __shared__ alignas(16) " << storage_ctype(objs[o].format) << " ro" << o << "["
                 << rw(static_cast<int>(o)) * rh(static_cast<int>(o)) << "];\n";
    // region inputs staged once: entry = input at the CLAMPED position
    bool staged = false;
    for (std::size_t o = 0; o < objs.size(); ++o) {
        if (objs[o].load < 0) continue;
        staged = true;
        const int f = field_in(objs[o].load);
        const char* ct = storage_ctype(objs[o].format);
        const int RWo = rw(static_cast<int>(o)), RHo = rh(static_cast<int>(o));
        const int co = colofs(static_cast<int>(o)), es = bytes_per_pixel(objs[o].format);
        const bool vec = vec_on && es <= 16 && 16 % es == 0 && (co * es) % 16 == 0 && (TW * es) % 16 == 0;
        if (vec) {
            // interior tiles: 16-byte copies of whole padded rows (the origin
            // column tx0 - co is 16-byte aligned: tx0 is a multiple of 32)
            const int vrow = RWo * es / 16; // uint4 per row
            body << "  if (tx0 - " << co << " >= 0 && ty0 - " << objs[o].halo_y << " >= 0 && tx0 + " << TW + co
                 << " <= W && ty0 + " << TH + objs[o].halo_y << " <= H && ty0 + " << TH << " <= ROW1 && ((p.f[" << f
                 << "] | p.f[" << f + 1 << "] | p.f[" << f + 2 << "]) & 15) == 0) {\n"
                 << "    for (int i = threadIdx.y * 32 + threadIdx.x; i < " << vrow * RHo << "; i += 256) {\n"
                 << "      const int ry = i / " << vrow << ", vx = i - ry * " << vrow << ";\n"
                 << "      const uint4* src = (const uint4*)((const unsigned char*)p.f[" << f << "] + (u64)fr * p.f[" << f + 2
                 << "] + (u64)(ty0 - " << objs[o].halo_y << " + ry) * p.f[" << f + 1 << "] + (u64)(tx0 - " << co << ") * "
                 << es << ");\n"
                 << "      reinterpret_cast<uint4*>(ro" << o << ")[i] = src[vx];\n"
                 << "    }\n  } else {\n";
        }
        // one row pointer per entry row; 32-column blocks unrolled
        body << "#pragma unroll\n  for (int ry = threadIdx.y, iy_ = 0; iy_ < " << (RHo + 7) / 8 << "; ++iy_, ry += 8) {\n"
             << (RHo % 8 ? "    if (ry >= " + std::to_string(RHo) + ") break;\n" : std::string())
             << "    const int y = clampi(ty0 - " << objs[o].halo_y << " + ry, max(0, ROW0 - " << objs[o].halo_y
             << "), min(H, ROW1 + " << objs[o].halo_y << ") - 1);\n"
             << "    const " << ct << "* src = (const " << ct << "*)((const unsigned char*)p.f[" << f << "] + (u64)fr * p.f["
             << f + 2 << "] + (u64)y * p.f[" << f + 1 << "]);\n"
             << "#pragma unroll\n    for (int ix = 0; ix < " << (RWo + 31) / 32 << "; ++ix) {\n"
             << "      const int rx = threadIdx.x + 32 * ix;\n" << (RWo % 32 ? "      if (rx >= " + std::to_string(RWo) + ") break;\n" : std::string())
             << "      ro" << o << "[ry * " << RWo << " + rx] = src[clampi(tx0 - " << colofs(static_cast<int>(o))
             << " + rx, 0, W - 1)];\n    }\n  }\n";
        if (vec) body << "  }\n";
    }
    if (staged) body << "  __syncthreads();\n";
    std::size_t tab_bytes = 0;
    std::size_t rs_bytes = 0; // separable row-sum buffer (declared at the top once its size is known)
    body << "@RSBUF@";
    for (std::size_t ni = 0; ni < nodes.size(); ++ni) {
        const RegionNode& rn = nodes[ni];
        const AbstractionKernel& k = *rn.k;
        std::vector<SlotInfo> no_outs;
        Emitter em(rn.in_slots, no_outs);
        em.prefix = "N" + std::to_string(ni) + "_";
        em.slot_obj = rn.in_obj;
        em.slot_param.resize(rn.in_param.size());
        for (std::size_t i = 0; i < rn.in_param.size(); ++i) em.slot_param[i] = rn.in_param[i] < 0 ? 0 : rn.in_param[i];
        em.obj_entry = entry;
        em.obj_type = otype;
        // outputs of this node (all share one region: the largest halo)
        int oref = -1;
        for (int o : rn.out_obj)
            if (o >= 0 && (oref < 0 || objs[static_cast<std::size_t>(o)].halo_x > objs[static_cast<std::size_t>(oref)].halo_x ||
                           objs[static_cast<std::size_t>(o)].halo_y > objs[static_cast<std::size_t>(oref)].halo_y))
                oref = o;
        if (oref < 0) throw unsupported("node without a region output");
        const RegionObject& R = objs[static_cast<std::size_t>(oref)];
        // a point node whose outputs are read only at the same entry by later
        // nodes of the region (no halo, not stored) and whose body cannot
        // raise (no division / array index) is not given a pass of its own:
        // its consumers evaluate its expression in place
        if (inline_node[ni]) {
            const PointKernel& pk = k.point();
            bool ok = true;
            {
                em.mode = Emitter::Mode::Point;
                std::vector<std::pair<int, Emitter::TV>> vals;
                for (std::size_t j = 0; j < rn.out_obj.size() && ok; ++j) {
                    if (rn.out_obj[j] < 0) continue;
                    std::fill(used_obj.begin(), used_obj.end(), false);
                    Emitter::TV v;
                    ok = em.temit(*pk.outputs[j].channel_bodies[0], v);
                    if (!ok) break;
                    const int o = rn.out_obj[j];
                    std::vector<int> uses;
                    for (std::size_t u = 0; u < objs.size(); ++u)
                        if (used_obj[u]) uses.push_back(static_cast<int>(u));
                    inline_uses[static_cast<std::size_t>(o)] = uses;
                    vals.push_back({o, v});
                }
                if (ok) {
                    for (auto& [o, v] : vals) {
                        TVproto& r = orange[static_cast<std::size_t>(o)];
                        if (v.t != 'd' && r.t != 'd' && v.lo >= r.lo && v.hi <= r.hi)
                            r.lo = static_cast<long long>(v.lo), r.hi = static_cast<long long>(v.hi);
                        const ImageFormat f = objs[static_cast<std::size_t>(o)].format;
                        inline_code[static_cast<std::size_t>(o)] =
                            f == ImageFormat::F32 ? "((float)" + Emitter::as_dbl(v) + ")"
                                                  : (v.t == 'd' ? std::string("0")
                                                                : "((" + std::string(storage_ctype(f)) + ")(" + v.c + "))");
                    }
                    body << "  // node " << ni << ": " << k.name << " (evaluated by its consumers)\n";
                    helpers << em.helpers.str();
                    std::fill(used_obj.begin(), used_obj.end(), false);
                    continue;
                }
            }
            throw unsupported("run-time typed point body");
        }
        // in-image entries only (their taps then sit at constant offsets from
        // the entry); out-of-image entries replicate the clamped one below
        std::ostringstream nb;
        std::string extra_base; // per-entry index of a tabulated tap array
        std::fill(used_obj.begin(), used_obj.end(), false);
        auto put = [&](int o, const Emitter::TV& v) {
            if (v.t != 'd' && orange[static_cast<std::size_t>(o)].t != 'd') {
                TVproto& r = orange[static_cast<std::size_t>(o)];
                if (v.lo >= r.lo && v.hi <= r.hi) r.lo = static_cast<long long>(v.lo), r.hi = static_cast<long long>(v.hi);
            }
            const ImageFormat f = objs[static_cast<std::size_t>(o)].format;
            std::string val;
            if (f == ImageFormat::F32) val = "(float)" + Emitter::as_dbl(v);
            else val = v.t == 'd' ? std::string("0") : "(" + std::string(storage_ctype(f)) + ")(" + v.c + ")";
            // every output entry of this node at the entry's position (a
            // smaller-halo output covers a sub-rectangle of the reference one)
            const RegionObject& O = objs[static_cast<std::size_t>(o)];
            if (O.halo_x == R.halo_x && O.halo_y == R.halo_y) {
                nb << "    ro" << o << "[e] = " << val << ";\n";
            } else {
                nb << "    { const int ox = rx - " << R.halo_x - O.halo_x << ", oy = ry - " << R.halo_y - O.halo_y
                   << "; if (ox >= 0 && oy >= 0 && ox < " << rw(o) << " && oy < " << rh(o) << ") ro" << o
                   << "[oy * " << rw(o) << " + ox] = " << val << "; }\n";
            }
        };
        if (k.kind == AbstractionKind::Point) {
            const PointKernel& pk = k.point();
            em.mode = Emitter::Mode::Point;
            for (std::size_t j = 0; j < rn.out_obj.size() && j < pk.outputs.size(); ++j) {
                if (rn.out_obj[j] < 0) continue;
                if (pk.outputs[j].channel_bodies.size() != 1) throw unsupported("multi-channel point output");
                Emitter::TV v;
                if (!em.temit(*pk.outputs[j].channel_bodies[0], v)) throw unsupported("run-time typed point body");
                put(rn.out_obj[j], v);
            }
        } else if (k.kind == AbstractionKind::Local) {
            const LocalKernel& lk = k.local();
            if (lk.median3x3) throw unsupported("median");
            em.local = &lk;
            em.mask = lk.mask.empty() ? &rn.matrix : &lk.mask;
            em.mode = Emitter::Mode::Tap;
            const int hw = lk.window_w / 2, hh = lk.window_h / 2;
            const Expr* mc = nullptr;
            const Expr* gexp = tab[ni] ? tabulated_g(lk, &mc) : nullptr;
            bool sep_box = !uses_op(*lk.tap_body, ExprOp::MaskCoef);
            if (!sep_box) { // a mask whose coefficients are all integer 1
                const std::vector<Value>& mk = lk.mask.empty() ? rn.matrix : lk.mask;
                sep_box = mk.size() == static_cast<std::size_t>(lk.window_w * lk.window_h);
                for (const Value& v : mk) sep_box = sep_box && !v.real && v.i == 1;
            }
            static const bool sep_on = std::getenv("GVX_REGION_NOSEP") == nullptr;
            sep_box = sep_box && sep_on;
            std::vector<Emitter::TV> gtaps;
            if (gexp) {
                // g once per position of the node's region + its window radius
                const int GW = rw(oref) + 2 * hw, GH = rh(oref) + 2 * hh;
                const std::string gx0 = "(tx0 - " + std::to_string(R.halo_x + hw) + ")",
                                  gy0 = "(ty0 - " + std::to_string(R.halo_y + hh) + ")";
                em.mode = Emitter::Mode::Tap;
                em.tdx = em.tdy = 0;
                std::fill(used_obj.begin(), used_obj.end(), false);
                Emitter::TV gv;
                if (!em.temit(*gexp, gv)) throw unsupported("run-time typed tap computation");
                const char* gty = gv.t == 'd' ? "double" : gv.t == 'l' ? "i64" : "int";
                const std::string ga = "gk" + std::to_string(ni);
                tab_bytes += static_cast<std::size_t>(GW) * GH * (gv.t == 'd' || gv.t == 'l' ? 8 : 4);
                body << "  // node " << ni << " tap computation, tabulated\n"
                     << "  __shared__ " << gty << " " << ga << "[" << GW * GH << "];\n"
                     << "  #pragma unroll\n  for (int ry = threadIdx.y, iy_ = 0; iy_ < " << (GH + 7) / 8 << "; ++iy_, ry += 8)\n"
                     << "  #pragma unroll\n"
                     << "  for (int ix = 0; ix < " << ((GW) + 31) / 32 << "; ++ix) {\n"
                     << (GH % 8 ? "    if (ry >= " + std::to_string(GH) + ") break;\n" : std::string())
                     << "    const int rx = threadIdx.x + 32 * ix;\n"
                     << "    if (rx >= " << (GW) << ") break;\n"
                     << "    const int e = ry * " << (GW) << " + rx;\n"
                     << "    const int px = " << gx0 << " + rx, py = " << gy0 << " + ry;\n";
                if (lk.boundary == BoundaryMode::Undefined)
                    body << "    if (px < 0 || py < 0 || px >= W || py >= H) continue;\n";
                else
                    body << "    if (px < -" << hw << " || py < -" << hh << " || px >= W + " << hw << " || py >= H + "
                         << hh << ") continue;\n";
                for (std::size_t o = 0; o < objs.size(); ++o)
                    if (used_obj[o])
                        body << "    const int b" << o << " = (py - ty0 + " << objs[o].halo_y << ") * "
                             << rw(static_cast<int>(o)) << " + px - tx0 + " << colofs(static_cast<int>(o)) << ";\n";
                body << "    " << ga << "[e] = (" << gty << ")(" << gv.c << ");\n  }\n  __syncthreads();\n";
                std::fill(used_obj.begin(), used_obj.end(), false);
                extra_base = "    const int bG = (py - " + gy0 + ") * " + std::to_string(GW) + " + px - " + gx0 + ";\n";
                const std::vector<Value>& mask = lk.mask.empty() ? rn.matrix : lk.mask;
                for (int dy = -hh; dy <= hh; ++dy)
                    for (int dx = -hw; dx <= hw; ++dx) {
                        Emitter::TV gt = gv;
                        gt.c = ga + "[bG + (" + std::to_string(dy * GW + dx) + ")]";
                        if (!mc) {
                            gtaps.push_back(gt);
                            continue;
                        }
                        const std::size_t mi = static_cast<std::size_t>((dy + hh) * lk.window_w + dx + hw);
                        if (mi >= mask.size()) throw unsupported("mask size");
                        const Emitter::TV cf = Emitter::tvalue(mask[mi]);
                        if (mask[mi].real || gt.t == 'd') {
                            gtaps.push_back(Emitter::tdbl("__dmul_rn(" + Emitter::as_dbl(cf) + ", " + Emitter::as_dbl(gt) + ")"));
                        } else {
                            const __int128 pr[4] = {cf.lo * gt.lo, cf.lo * gt.hi, cf.hi * gt.lo, cf.hi * gt.hi};
                            gtaps.push_back(Emitter::tbin_int("*", cf, gt, std::min({pr[0], pr[1], pr[2], pr[3]}),
                                                              std::max({pr[0], pr[1], pr[2], pr[3]})));
                        }
                    }
            }
            if (lk.boundary == BoundaryMode::Undefined) {
                Emitter::TV z = Emitter::tint("0", 0, 0);
                nb << "    if (px < " << hw << " || py < " << hh << " || px >= W - " << hw << " || py >= H - " << hh
                     << ") {\n";
                for (int o : rn.out_obj)
                    if (o >= 0) put(o, z);
                nb << "      continue;\n    }\n";
            }
            em.mode = Emitter::Mode::Tap;
            // separable evaluation of box-like sums (Clamp border, integer taps
            // whose mask coefficients are all 1, no wrapping): each row of the
            // window summed once per position into shared memory, then the
            // rows of the window summed per entry -- w + h - 1 instead of w h
            // tap evaluations per entry
            std::string taps;
            if (!gexp && sep_box && lk.combine == CombineMode::Sum && lk.boundary == BoundaryMode::Clamp && hh > 0) {
                std::vector<Emitter::TV> row;
                bool ok = true;
                std::fill(used_obj.begin(), used_obj.end(), false);
                for (int dx = -hw; dx <= hw && ok; ++dx) {
                    em.tdx = dx;
                    em.tdy = 0;
                    Emitter::TV t;
                    ok = em.temit(*lk.tap_body, t) && t.t != 'd';
                    row.push_back(t);
                }
                __int128 lo = 0, hi = 0;
                for (const Emitter::TV& t : row) lo += t.lo, hi += t.hi;
                const __int128 tlo = lo * lk.window_h, thi = hi * lk.window_h;
                ok = ok && tlo >= Emitter::kI64Lo && thi <= Emitter::kI64Hi;
                if (ok) {
                    const bool i32 = tlo >= Emitter::kI32Lo && thi <= Emitter::kI32Hi;
                    const char* ty = i32 ? "int" : "i64";
                    const int RW = rw(oref), RHs = rh(oref) + 2 * hh;
                    const std::string rs = "rs" + std::to_string(ni);
                    std::ostringstream sum;
                    for (std::size_t k = 0; k < row.size(); ++k)
                        sum << (k ? " + " : "") << (i32 ? row[k].c : Emitter::as_i64(row[k]));
                    rs_bytes = std::max(rs_bytes, static_cast<std::size_t>(RW) * RHs * (i32 ? 4 : 8));
                    body << "  // node " << ni << ": window rows summed once per position\n"
                         << "  " << ty << "* " << rs << " = reinterpret_cast<" << ty << "*>(rsbuf);\n"
                         << "  #pragma unroll\n  for (int ry = threadIdx.y, iy_ = 0; iy_ < " << (RHs + 7) / 8 << "; ++iy_, ry += 8)\n"
                         << "  #pragma unroll\n"
                         << "  for (int ix = 0; ix < " << (RW + 31) / 32 << "; ++ix) {\n"
                         << (RHs % 8 ? "    if (ry >= " + std::to_string(RHs) + ") break;\n" : std::string())
                         << "    const int rx = threadIdx.x + 32 * ix;\n";
                    if (RW % 32) body << "    if (rx >= " << RW << ") break;\n";
                    body << "    const int px = tx0 - " << R.halo_x << " + rx, py = ty0 - " << R.halo_y + hh << " + ry;\n";
                    for (std::size_t o = 0; o < objs.size(); ++o)
                        if (used_obj[o])
                            body << "    const int b" << o << " = (py - ty0 + " << objs[o].halo_y << ") * "
                                 << rw(static_cast<int>(o)) << " + px - tx0 + " << colofs(static_cast<int>(o)) << ";\n";
                    body << "    " << rs << "[ry * " << RW << " + rx] = (" << ty << ")(" << sum.str() << ");\n"
                         << "  }\n  __syncthreads();\n";
                    // per entry: the window's rows (entry rows ry .. ry + 2 hh of rs)
                    std::ostringstream cs;
                    cs << "    " << ty << " cmbt = " << rs << "[(ry + 0) * " << RW << " + rx]";
                    for (int dy = 1; dy < lk.window_h; ++dy) cs << " + " << rs << "[(ry + " << dy << ") * " << RW << " + rx]";
                    cs << ";\n    V cmb = vi((i64)cmbt);\n";
                    taps = cs.str();
                    Emitter::TV acc = Emitter::tint("cmbt", lo * lk.window_h, hi * lk.window_h);
                    if (!i32) acc.t = 'l';
                    em.cmb_typed = true;
                    em.cmb_tv = acc;
                    std::fill(used_obj.begin(), used_obj.end(), false);
                }
            }
            if (taps.empty()) taps = gexp ? typed_combine(em, lk, gtaps) : typed_taps(em, lk);
            if (taps.empty()) throw unsupported("run-time typed tap body");
            em.tdx = em.tdy = 0;
            em.mode = Emitter::Mode::Post;
            Emitter::TV v = em.cmb_tv;
            if (lk.post_body && !em.temit(*lk.post_body, v)) throw unsupported("run-time typed post body");
            nb << taps;
            for (int o : rn.out_obj)
                if (o >= 0) put(o, v);
        } else {
            throw unsupported("node kind");
        }
        // two copies of the entry loop: tiles whose node region lies inside
        // the image skip the per-entry position test
        std::ostringstream bases;
        for (std::size_t o = 0; o < objs.size(); ++o)
            if (used_obj[o])
                bases << "    const int b" << o << " = (py - ty0 + " << objs[o].halo_y << ") * " << rw(static_cast<int>(o))
                      << " + px - tx0 + " << colofs(static_cast<int>(o)) << ";\n";
        body << "  // node " << ni << ": " << k.name << "\n";
        for (int border = 0; border < 2; ++border) {
            if (border == 0)
                body << "  if (tx0 - " << R.halo_x << " >= 0 && ty0 - " << R.halo_y << " >= 0 && tx0 + " << TW + R.halo_x
                     << " <= W && ty0 + " << TH + R.halo_y << " <= H) {\n";
            else
                body << "  } else {\n";
            body << "  #pragma unroll\n  for (int ry = threadIdx.y, iy_ = 0; iy_ < " << (rh(oref) + 7) / 8 << "; ++iy_, ry += 8)\n"
                 << "  #pragma unroll\n"
                 << "  for (int ix = 0; ix < " << (rw(oref) + 31) / 32 << "; ++ix) {\n"
                 << (rh(oref) % 8 ? "    if (ry >= " + std::to_string(rh(oref)) + ") break;\n" : std::string())
                 << "    const int rx = threadIdx.x + 32 * ix;\n";
            if (rw(oref) % 32) body << "    if (rx >= " << rw(oref) << ") break;\n";
            body << "    const int e = ry * " << rw(oref) << " + rx;\n"
                 << "    const int px = tx0 - " << R.halo_x << " + rx, py = ty0 - " << R.halo_y << " + ry;\n";
            if (border) body << "    if (px < 0 || py < 0 || px >= W || py >= H) continue;\n";
            body << bases.str() << extra_base << nb.str() << "  }\n";
        }
        body << "  }\n  __syncthreads();\n";
        // out-of-image entries = the entry at the clamped position (border
        // tiles); an object without halo is only ever read at in-image entries
        for (int o : rn.out_obj) {
            if (o < 0) continue;
            const RegionObject& O = objs[static_cast<std::size_t>(o)];
            if (O.halo_x == 0 && O.halo_y == 0) continue;
            body << "  if (tx0 - " << O.halo_x << " < 0 || ty0 - " << O.halo_y << " < 0 || tx0 + " << TW + O.halo_x
                 << " > W || ty0 + " << TH + O.halo_y << " > H) {\n"
                 << "    #pragma unroll\n    for (int ry = threadIdx.y, iy_ = 0; iy_ < " << (rh(o) + 7) / 8 << "; ++iy_, ry += 8)\n"
                 << "    #pragma unroll\n"
                 << "    for (int ix = 0; ix < " << ((rw(o)) + 31) / 32 << "; ++ix) {\n"
                 << (rh(o) % 8 ? "      if (ry >= " + std::to_string(rh(o)) + ") break;\n" : std::string())
                 << "      const int rx = threadIdx.x + 32 * ix;\n"
                 << "      if (rx >= " << (rw(o)) << ") break;\n"
                 << "      const int e = ry * " << (rw(o)) << " + rx;\n"
                 << "      const int x = tx0 - " << O.halo_x << " + rx, y = ty0 - " << O.halo_y << " + ry;\n"
                 << "      if (x >= 0 && y >= 0 && x < W && y < H) continue;\n"
                 << "      ro" << o << "[e] = ro" << o << "[(clampi(y, 0, H - 1) - ty0 + " << O.halo_y << ") * " << rw(o)
                 << " + clampi(x, 0, W - 1) - tx0 + " << O.halo_x << "];\n    }\n    __syncthreads();\n  }\n";
        }
        // per-node helper functions (typed loaders of global inputs)
        std::string h = em.helpers.str();
        helpers << h;
    }
    // stores of the objects consumed outside the region (or observable)
    for (std::size_t o = 0; o < objs.size(); ++o) {
        if (objs[o].store < 0) continue;
        const int f = field_in(static_cast<int>(ins.size()) + objs[o].store);
        const char* ct = storage_ctype(objs[o].format);
        const int es = bytes_per_pixel(objs[o].format), RWs = rw(static_cast<int>(o));
        const bool vec = vec_on && es <= 16 && 16 % es == 0 && (objs[o].halo_x * es) % 16 == 0 && (RWs * es) % 16 == 0 &&
                         (TW * es) % 16 == 0;
        if (vec) { // interior tiles: 16-byte copies of whole tile rows
            const int vrow = TW * es / 16;
            body << "  if (tx0 + " << TW << " <= W && ty0 + " << TH << " <= ROW1 && ((p.f[" << f << "] | p.f[" << f + 1
                 << "] | p.f[" << f + 2 << "]) & 15) == 0) {\n"
                 << "    for (int i = threadIdx.y * 32 + threadIdx.x; i < " << vrow * TH << "; i += 256) {\n"
                 << "      const int ry = i / " << vrow << ", vx = i - ry * " << vrow << ";\n"
                 << "      uint4* dst = (uint4*)((unsigned char*)p.f[" << f << "] + (u64)fr * p.f[" << f + 2
                 << "] + (u64)(ty0 + ry) * p.f[" << f + 1 << "] + (u64)tx0 * " << es << ");\n"
                 << "      dst[vx] = reinterpret_cast<const uint4*>(ro" << o << " + (ry + " << objs[o].halo_y << ") * " << RWs
                 << " + " << objs[o].halo_x << ")[vx];\n"
                 << "    }\n  } else {\n";
        }
        body << "#pragma unroll\n  for (int ry = threadIdx.y, iy_ = 0; iy_ < " << (TH + 7) / 8 << "; ++iy_, ry += 8) {\n"
             << "    const int gy = ty0 + ry;\n    if (gy >= ROW1) break;\n"
             << "    " << ct << "* row = (" << ct << "*)((unsigned char*)p.f[" << f << "] + (u64)fr * p.f[" << f + 2
             << "] + (u64)gy * p.f[" << f + 1 << "]);\n"
             << "#pragma unroll\n    for (int ix = 0; ix < " << TW / 32 << "; ++ix) {\n"
             << "      const int rx = threadIdx.x + 32 * ix, gx = tx0 + rx;\n      if (gx >= W) break;\n"
             << "      row[gx] = ro" << o << "[(ry + " << objs[o].halo_y << ") * " << rw(static_cast<int>(o)) << " + rx + "
             << objs[o].halo_x << "];\n    }\n  }\n";
        if (vec) body << "  }\n";
    }
    body << "  (void)rd;\n}\n";
    KernelSpec ks;
    ks.name = "gvx_region";
    ks.grid = KernelSpec::Grid::Pixels;
    ks.block_x = 32;
    ks.block_y = 8;
    ks.cols = TW / 32;
    ks.rows = TH / 8;
    std::string pre = kPrelude;
    const std::string key = "NFIELDS";
    pre.replace(pre.find(key), key.size(), std::to_string(prog.fields()));
    smem = tab_bytes + rs_bytes;
    for (std::size_t o = 0; o < objs.size(); ++o)
        if (!inline_obj[o])
            smem += static_cast<std::size_t>(rw(static_cast<int>(o))) * rh(static_cast<int>(o)) *
                    static_cast<std::size_t>(bytes_per_pixel(objs[o].format));
    std::string text = body.str();
    const std::size_t at = text.find("@RSBUF@");
    text.replace(at, 7, rs_bytes ? "  __shared__ alignas(8) unsigned char rsbuf[" + std::to_string(rs_bytes) + "];\n" : "");
    ks.source = pre + helpers.str() + text;
    prog.kernels.push_back(std::move(ks));
    return prog;
}

} // namespace

NodeProgram lower_region(const std::vector<RegionNode>& nodes, const std::vector<RegionObject>& objs,
                         const std::vector<SlotInfo>& ins, const std::vector<SlotInfo>& outs) {
    // 128 x 16 outputs per 256-thread block (measured against 64 x 16 / 64 x 32
    // / 128 x 8 / 32 x 32: sobel.json 382 -> 431, laplacian.json 646 -> 849
    // Gpx/s), halved while the emitted kernel's shared memory exceeds 36 KB
    // (harris.json / tomasi.json: 128 x 8 at 22 KB beat 128 x 16 at 38 KB,
    // 164 vs 160 Gpx/s: more resident blocks)
    int TW = 128, TH = 16;
    if (const char* e = std::getenv("GVX_REGION_TW")) TW = std::max(32, std::atoi(e) / 32 * 32); // tuning experiments
    if (const char* e = std::getenv("GVX_REGION_TH")) TH = std::max(8, std::atoi(e) / 8 * 8);
    static const std::size_t cap = [] {
        const char* e = std::getenv("GVX_REGION_SMEM_KB"); // tuning experiments
        return static_cast<std::size_t>(std::min(e ? std::atoi(e) : 36, 46)) * 1024;
    }();
    for (;;) {
        std::size_t smem = 0;
        NodeProgram prog = lower_region_at(nodes, objs, ins, outs, TW, TH, smem);
        if (smem <= cap) return prog;
        if (TW <= 32 && TH <= 8) throw Error(ErrorCode::UnsupportedKind, "region: intermediates exceed shared memory");
        (TH > 8 ? TH : TW) /= 2;
    }
}

NodeProgram lower_node(const AbstractionKernel& k, const std::vector<SlotInfo>& ins,
                       const std::vector<SlotInfo>& outs, const std::vector<Value>& matrix_values,
                       bool count_reads) {
    NodeProgram p;
    switch (k.kind) {
    case AbstractionKind::Point: p = lower_point(k, ins, outs, /*vector_io=*/!count_reads); break;
    case AbstractionKind::Local:
        if (!count_reads && !std::getenv("GVX_NO_LTILE")) p = lower_local_tiled(k, ins, outs, matrix_values);
        if (p.kernels.empty()) p = lower_local(k, ins, outs, matrix_values);
        break;
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
