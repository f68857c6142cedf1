// fft.cuh -- FP64 negacyclic transform for N = 1024 (512 complex points), one
// 64-thread group per polynomial, 8 complex points per thread in registers.
//
// The arithmetic is the contract stated in oracle/tfhe_oracle.c (the oracle's
// FFT mode executes the same operations in the same order, so the GPU is bit-exact
// with it):
//
//   forward  a_j = d_j + i d_{j+512} (integer digits) -> Z_k = sum_j a_j psi^j W^{jk}
//            in slot bitrev9(k): Cooley-Tukey with the negacyclic twist absorbed into
//            the twiddles (tree node v = 2^s + b at stage s has twiddle psi^(E[v]/2),
//            E[1] = 512, children E/2 and E/2 + 1024 mod 2048).  No twist multiply.
//   inverse  plain inverse DFT, radix-2 DIT, bit-reversed in -> natural out; the
//            untwist conj(psi^j) is applied by the caller; 1/512 lives in the BK.
//
// Butterflies (every op is an __*_rn intrinsic, so nvcc cannot contract or reorder):
//   ct<ROT>(u, v, w)  w = (c, t) stands for c (1 + i t); v is first rotated by
//                     ROT (0: none, 1: i, 3: -i, exact); s = (fma(-vi, t, vr),
//                     fma(vr, t, vi)); u' = u + c s, v' = u - c s as fmas.
//                     6 DFMA instead of the 8 FP64 ops of a complex-multiply butterfly.
//   std_(u, v, w)     t = cmul(v, w); u' = u + t; v' = u - t (8 ops) -- used where the
//                     per-thread twiddle can be exactly -i (first stage of an inverse
//                     pass), for which (c, t) is degenerate.
//   bf_1 / bf_mi      w = 1 / w = -i: four adds.
// A stage's twiddle is a per-thread register value at the first stage of each
// register pass (its index bits are thread bits) and a register value times a
// compile-time rotation at the other two stages (the sibling bit is a register bit).
//
// Register layouts (M = 512, thread t in [0, 64), t = 8k + r):
//   pass 0 : x[q] = position t + 64 q        (natural order: the folded input)
//   pass 1 : x[m] = position 64 k + 8 m + r
//   pass 2 : x[q] = position 8 t + q         (bit-reversed order: frequency slots)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lpb {

constexpr int FFT_THREADS = 64;
constexpr int FFT_M = 512;

__device__ __forceinline__ double2 cmul(double2 a, double2 w)
{
    double2 r;
    r.x = __fma_rn(a.x, w.x, -__dmul_rn(a.y, w.y));
    r.y = __fma_rn(a.x, w.y, __dmul_rn(a.y, w.x));
    return r;
}
__device__ __forceinline__ double2 conj2(double2 w) { return make_double2(w.x, -w.y); }

template <int ROT>
__device__ __forceinline__ void ct(double2& u, double2& v, double2 w)
{
    double xr, xi;
    if constexpr (ROT == 0) {
        xr = v.x;
        xi = v.y;
    } else if constexpr (ROT == 1) {  // i v
        xr = -v.y;
        xi = v.x;
    } else {  // -i v
        xr = v.y;
        xi = -v.x;
    }
    const double sr = __fma_rn(-xi, w.y, xr);
    const double si = __fma_rn(xr, w.y, xi);
    const double a = u.x, b = u.y;
    u.x = __fma_rn(w.x, sr, a);
    u.y = __fma_rn(w.x, si, b);
    v.x = __fma_rn(-w.x, sr, a);
    v.y = __fma_rn(-w.x, si, b);
}
__device__ __forceinline__ void std_(double2& u, double2& v, double2 w)
{
    const double2 tt = cmul(v, w);
    const double a = u.x, b = u.y;
    u.x = __dadd_rn(a, tt.x);
    u.y = __dadd_rn(b, tt.y);
    v.x = __dsub_rn(a, tt.x);
    v.y = __dsub_rn(b, tt.y);
}
__device__ __forceinline__ void bf_1(double2& u, double2& v)
{
    const double2 a = u, c = v;
    u = make_double2(__dadd_rn(a.x, c.x), __dadd_rn(a.y, c.y));
    v = make_double2(__dsub_rn(a.x, c.x), __dsub_rn(a.y, c.y));
}
__device__ __forceinline__ void bf_mi(double2& u, double2& v)  // w = -i: -i v = (vi, -vr)
{
    const double2 a = u;
    const double c = v.y, d = -v.x;
    u = make_double2(__dadd_rn(a.x, c), __dadd_rn(a.y, d));
    v = make_double2(__dsub_rn(a.x, c), __dsub_rn(a.y, d));
}

// Exchange tile layout: position 64k + 8m + r (k, m, r in [0, 8)) lives at slot
// 72k + 9m + r (576 slots).  Every register layout then addresses its 8 elements as
// base + constant (72 q, 9 m or r), and each quarter warp (8 lanes x 16 B) hits 8
// distinct 16-byte bank groups in all three layouts: conflict-free.
constexpr int XTILE = 576;
__device__ __forceinline__ int slot_of(int k, int m, int r) { return 72 * k + 9 * m + r; }

// Per-thread twiddles.  Host tables (engine.cu make_tables) hold them per thread,
// [entry][t], so a CTA loads them with coalesced 16-byte loads.
constexpr int TW_ENTRIES = 8;
struct FwdTw {  // (c, tan): stage 3, 4, 5 (2), 6, 7, 8 (2)
    double2 s3, s4, s5a, s5b, s6, s7, s8a, s8b;
};
struct InvTw {  // h = 8 (std, conj W), 16, 32 (2) | h = 64 (std, conj W), 128, 256 (2)
    double2 h8, h16, h32a, h32b, h64, h128, h256a, h256b;
};
// pass-0 forward twiddles are the same for every thread: nodes 1, 2, 4, 6 (c, tan)
__constant__ double2 c_fwd0[4];
// inverse h = 4 base (cos, -tan) of W^64 (conjugated)
__constant__ double2 c_inv4;

__device__ __forceinline__ FwdTw load_fwd_tw(const double2* __restrict__ T, int t)
{
    FwdTw w;
    w.s3 = T[0 * 64 + t];
    w.s4 = T[1 * 64 + t];
    w.s5a = T[2 * 64 + t];
    w.s5b = T[3 * 64 + t];
    w.s6 = T[4 * 64 + t];
    w.s7 = T[5 * 64 + t];
    w.s8a = T[6 * 64 + t];
    w.s8b = T[7 * 64 + t];
    return w;
}
__device__ __forceinline__ InvTw load_inv_tw(const double2* __restrict__ T, int t)
{
    InvTw w;
    w.h8 = __ldg(T + 0 * 64 + t);
    w.h16 = __ldg(T + 1 * 64 + t);
    w.h32a = __ldg(T + 2 * 64 + t);
    w.h32b = __ldg(T + 3 * 64 + t);
    w.h64 = __ldg(T + 4 * 64 + t);
    w.h128 = __ldg(T + 5 * 64 + t);
    w.h256a = __ldg(T + 6 * 64 + t);
    w.h256b = __ldg(T + 7 * 64 + t);
    return w;
}

// ---- forward passes (tree stages 0-2, 3-5, 6-8)
__device__ __forceinline__ void fwd_pass0(double2 x[8])
{
    const double2 n1 = c_fwd0[0], n2 = c_fwd0[1], n4 = c_fwd0[2], n6 = c_fwd0[3];
    ct<0>(x[0], x[4], n1);
    ct<0>(x[1], x[5], n1);
    ct<0>(x[2], x[6], n1);
    ct<0>(x[3], x[7], n1);
    ct<0>(x[0], x[2], n2);
    ct<0>(x[1], x[3], n2);
    ct<1>(x[4], x[6], n2);
    ct<1>(x[5], x[7], n2);
    ct<0>(x[0], x[1], n4);
    ct<1>(x[2], x[3], n4);
    ct<0>(x[4], x[5], n6);
    ct<1>(x[6], x[7], n6);
}
__device__ __forceinline__ void fwd_pass1(double2 x[8], const FwdTw& w)
{
    ct<0>(x[0], x[4], w.s3);
    ct<0>(x[1], x[5], w.s3);
    ct<0>(x[2], x[6], w.s3);
    ct<0>(x[3], x[7], w.s3);
    ct<0>(x[0], x[2], w.s4);
    ct<0>(x[1], x[3], w.s4);
    ct<1>(x[4], x[6], w.s4);
    ct<1>(x[5], x[7], w.s4);
    ct<0>(x[0], x[1], w.s5a);
    ct<1>(x[2], x[3], w.s5a);
    ct<0>(x[4], x[5], w.s5b);
    ct<1>(x[6], x[7], w.s5b);
}
__device__ __forceinline__ void fwd_pass2(double2 x[8], const FwdTw& w)
{
    ct<0>(x[0], x[4], w.s6);
    ct<0>(x[1], x[5], w.s6);
    ct<0>(x[2], x[6], w.s6);
    ct<0>(x[3], x[7], w.s6);
    ct<0>(x[0], x[2], w.s7);
    ct<0>(x[1], x[3], w.s7);
    ct<1>(x[4], x[6], w.s7);
    ct<1>(x[5], x[7], w.s7);
    ct<0>(x[0], x[1], w.s8a);
    ct<1>(x[2], x[3], w.s8a);
    ct<0>(x[4], x[5], w.s8b);
    ct<1>(x[6], x[7], w.s8b);
}

// ---- inverse passes (h = 1, 2, 4 | 8, 16, 32 | 64, 128, 256)
__device__ __forceinline__ void inv_pass2(double2 x[8])
{
    bf_1(x[0], x[1]);
    bf_1(x[2], x[3]);
    bf_1(x[4], x[5]);
    bf_1(x[6], x[7]);
    bf_1(x[0], x[2]);
    bf_mi(x[1], x[3]);
    bf_1(x[4], x[6]);
    bf_mi(x[5], x[7]);
    const double2 b = c_inv4;
    bf_1(x[0], x[4]);
    ct<0>(x[1], x[5], b);
    bf_mi(x[2], x[6]);
    ct<3>(x[3], x[7], b);
}
__device__ __forceinline__ void inv_pass1(double2 x[8], const InvTw& w)
{
    std_(x[0], x[1], w.h8);
    std_(x[2], x[3], w.h8);
    std_(x[4], x[5], w.h8);
    std_(x[6], x[7], w.h8);
    ct<0>(x[0], x[2], w.h16);
    ct<3>(x[1], x[3], w.h16);
    ct<0>(x[4], x[6], w.h16);
    ct<3>(x[5], x[7], w.h16);
    ct<0>(x[0], x[4], w.h32a);
    ct<0>(x[1], x[5], w.h32b);
    ct<3>(x[2], x[6], w.h32a);
    ct<3>(x[3], x[7], w.h32b);
}
__device__ __forceinline__ void inv_pass0(double2 x[8], const InvTw& w)
{
    std_(x[0], x[1], w.h64);
    std_(x[2], x[3], w.h64);
    std_(x[4], x[5], w.h64);
    std_(x[6], x[7], w.h64);
    ct<0>(x[0], x[2], w.h128);
    ct<3>(x[1], x[3], w.h128);
    ct<0>(x[4], x[6], w.h128);
    ct<3>(x[5], x[7], w.h128);
    ct<0>(x[0], x[4], w.h256a);
    ct<0>(x[1], x[5], w.h256b);
    ct<3>(x[2], x[6], w.h256a);
    ct<3>(x[3], x[7], w.h256b);
}

// Exchange helpers.  `bar` synchronises the threads that share the tile.
// pass-0 layout: thread t = 8m + r holds k = q;  pass-1: t = 8k + r holds m;
// pass-2: t = 8k + m holds r.
template <class Bar>
__device__ __forceinline__ void exch_p0_to_p1(double2 x[8], double2* buf, int t, Bar bar)
{
    double2* w = buf + slot_of(0, t >> 3, t & 7);
#pragma unroll
    for (int q = 0; q < 8; q++)
        w[72 * q] = x[q];
    bar();
    const double2* rd = buf + slot_of(t >> 3, 0, t & 7);
#pragma unroll
    for (int m = 0; m < 8; m++)
        x[m] = rd[9 * m];
}
template <class Bar>
__device__ __forceinline__ void exch_p1_to_p2(double2 x[8], double2* buf, int t, Bar bar)
{
    bar();  // the warp's previous reads of this single tile are done
    double2* w = buf + slot_of(t >> 3, 0, t & 7);
#pragma unroll
    for (int m = 0; m < 8; m++)
        w[9 * m] = x[m];
    bar();
    const double2* rd = buf + slot_of(t >> 3, t & 7, 0);
#pragma unroll
    for (int q = 0; q < 8; q++)
        x[q] = rd[q];
}

// Forward transform of the folded integer input x (pass-0 layout) -> frequency slots
// (pass-2 layout).  bufX: cross-warp exchange tile (needs the 64-thread barrier `bar`);
// bufW: intra-warp exchange tile (after tree stage 0 the two 256-point halves are
// independent and warp w owns half w in passes 1 and 2, so `wbar` = __syncwarp).
template <class Bar, class WBar>
__device__ __forceinline__ void fft_forward(double2 x[8], const FwdTw& tw, double2* bufX,
                                            double2* bufW, int t, Bar bar, WBar wbar)
{
    fwd_pass0(x);
    exch_p0_to_p1(x, bufX, t, bar);
    fwd_pass1(x, tw);
    exch_p1_to_p2(x, bufW, t, wbar);
    fwd_pass2(x, tw);
}

// Inverse transform (unscaled, no untwist) of frequency slots (pass-2 layout) ->
// natural order (pass-0 layout), for one polynomial.
template <class Bar, class WBar>
__device__ __forceinline__ void fft_inverse(double2 x[8], const InvTw& tw, double2* bufX,
                                            double2* bufW, int t, Bar bar, WBar wbar)
{
    inv_pass2(x);
    {
        wbar();
        double2* w = bufW + slot_of(t >> 3, t & 7, 0);
#pragma unroll
        for (int q = 0; q < 8; q++)
            w[q] = x[q];
        wbar();
        const double2* rd = bufW + slot_of(t >> 3, 0, t & 7);
#pragma unroll
        for (int m = 0; m < 8; m++)
            x[m] = rd[9 * m];
    }
    inv_pass1(x, tw);
    {
        bar();
        double2* w = bufX + slot_of(t >> 3, 0, t & 7);
#pragma unroll
        for (int m = 0; m < 8; m++)
            w[9 * m] = x[m];
        bar();
        const double2* rd = bufX + slot_of(0, t >> 3, t & 7);
#pragma unroll
        for (int q = 0; q < 8; q++)
            x[q] = rd[72 * q];
    }
    inv_pass0(x, tw);
}

// Two inverse transforms in lockstep (outputs A and B of one external product): they
// share every exchange barrier and the compiler interleaves their butterflies.
// c0/c1 cross tiles, w0/w1 intra tiles (may alias c0/c1: a CTA barrier separates uses).
template <class Bar, class WBar>
__device__ __forceinline__ void fft_inverse2(double2 x0[8], double2 x1[8], const InvTw& tw,
                                             double2* c0, double2* c1, double2* w0, double2* w1,
                                             int t, Bar bar, WBar wbar)
{
    inv_pass2(x0);
    inv_pass2(x1);
    {
        wbar();
        double2* a = w0 + slot_of(t >> 3, t & 7, 0);
        double2* b = w1 + slot_of(t >> 3, t & 7, 0);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            a[q] = x0[q];
            b[q] = x1[q];
        }
        wbar();
        const double2* ra = w0 + slot_of(t >> 3, 0, t & 7);
        const double2* rb = w1 + slot_of(t >> 3, 0, t & 7);
#pragma unroll
        for (int m = 0; m < 8; m++) {
            x0[m] = ra[9 * m];
            x1[m] = rb[9 * m];
        }
    }
    inv_pass1(x0, tw);
    inv_pass1(x1, tw);
    bar();
    {
        double2* a = c0 + slot_of(t >> 3, 0, t & 7);
        double2* b = c1 + slot_of(t >> 3, 0, t & 7);
#pragma unroll
        for (int m = 0; m < 8; m++) {
            a[9 * m] = x0[m];
            b[9 * m] = x1[m];
        }
        bar();
        const double2* ra = c0 + slot_of(0, t >> 3, t & 7);
        const double2* rb = c1 + slot_of(0, t >> 3, t & 7);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            x0[q] = ra[72 * q];
            x1[q] = rb[72 * q];
        }
    }
    inv_pass0(x0, tw);
    inv_pass0(x1, tw);
}

}  // namespace lpb
