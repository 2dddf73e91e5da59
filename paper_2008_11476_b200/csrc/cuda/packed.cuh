// Packed-FP32 helpers for the stencil kernels.
//
// Blackwell issues FP32 arithmetic at full rate only as packed pairs
// (FFMA2 / FADD2 / FMUL2 on register pairs).  The stencil kernels keep four
// adjacent columns of every quantity as an (even, odd) pair of float2 —
// columns (c, c+2) and (c+1, c+3) — so each separable 3-tap step
// (x[k-1], x[k], x[k+1]) combines register-aligned pairs:
//   P1 = (c-1, c+1)   P2 = (c, c+2)   P3 = (c+1, c+3)   P4 = (c+2, c+4)
// All values carried this way are integers < 2^24, i.e. exact in fp32.
#pragma once

#include "tile.cuh"

namespace gvxd {

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

/// 2^23 + byte k of w (the float bit pattern 0x4B0000bb).
__device__ __forceinline__ float magic_byte(uint32_t w, int k) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7440u | static_cast<unsigned>(k)));
}

/// Four columns as (even, odd) pairs.
struct Q4 {
    float2 e, o;
};
__device__ __forceinline__ Q4 qadd(Q4 a, Q4 b) { return Q4{add2(a.e, b.e), add2(a.o, b.o)}; }
__device__ __forceinline__ Q4 qsub(Q4 a, Q4 b) { return Q4{sub2(a.e, b.e), sub2(a.o, b.o)}; }
__device__ __forceinline__ Q4 qmul(Q4 a, Q4 b) { return Q4{mul2(a.e, b.e), mul2(a.o, b.o)}; }

/// Column pairs of source bytes c-1 .. c+4 around the aligned word at smem
/// offset `off`: (P1, P2, P3, P4) as exact floats.
struct Cols6 {
    float2 p1, p2, p3, p4;
};
__device__ __forceinline__ Cols6 load_cols6(const uint8_t* row, int off) {
    const uint32_t wl = lds32(row, off - 4), wc = lds32(row, off), wr = lds32(row, off + 4);
    const float2 magic = f2(-8388608.f, -8388608.f);
    Cols6 c;
    c.p1 = add2(f2(magic_byte(wl, 3), magic_byte(wc, 1)), magic);
    c.p2 = add2(f2(magic_byte(wc, 0), magic_byte(wc, 2)), magic);
    c.p3 = add2(f2(magic_byte(wc, 1), magic_byte(wc, 3)), magic);
    c.p4 = add2(f2(magic_byte(wc, 2), magic_byte(wr, 0)), magic);
    return c;
}

/// As load_cols6 with +2 on P1 and P4: the smooth terms S of both column
/// pairs come out biased by +2 (the differences D are then meaningless).
/// Used by the Gaussian so that the vertical 1-2-1 sum carries its +8
/// rounding bias for free.
__device__ __forceinline__ Cols6 load_cols6_biased(const uint8_t* row, int off) {
    const uint32_t wl = lds32(row, off - 4), wc = lds32(row, off), wr = lds32(row, off + 4);
    const float2 magic = f2(-8388608.f, -8388608.f), biased = f2(-8388606.f, -8388606.f);
    Cols6 c;
    c.p1 = add2(f2(magic_byte(wl, 3), magic_byte(wc, 1)), biased);
    c.p2 = add2(f2(magic_byte(wc, 0), magic_byte(wc, 2)), magic);
    c.p3 = add2(f2(magic_byte(wc, 1), magic_byte(wc, 3)), magic);
    c.p4 = add2(f2(magic_byte(wc, 2), magic_byte(wr, 0)), biased);
    return c;
}

/// Separable 3-tap terms of 4 columns from their 6-column neighbourhood:
/// D = x[k+1] - x[k-1] (Sobel-x row term), S = x[k-1] + 2 x[k] + x[k+1].
__device__ __forceinline__ void diff_smooth(const Cols6& c, Q4& D, Q4& S) {
    const float2 two = f2(2.f, 2.f);
    D = Q4{sub2(c.p3, c.p1), sub2(c.p4, c.p2)};
    S = Q4{fma2(two, c.p2, add2(c.p1, c.p3)), fma2(two, c.p3, add2(c.p2, c.p4))};
}

/// Rebuilds the 6-column neighbourhood of an in-register quantity q (4
/// columns) with its left / right neighbour columns from adjacent lanes.
__device__ __forceinline__ Cols6 neighbourhood(Q4 q, float left, float right) {
    Cols6 c;
    c.p1 = f2(left, q.o.x);
    c.p2 = q.e;
    c.p3 = q.o;
    c.p4 = f2(q.e.y, right);
    return c;
}

} // namespace gvxd
