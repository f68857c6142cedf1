// fft.cuh -- FP64 negacyclic transform for N = 1024 (512 complex points), one
// 64-thread group per polynomial, 8 complex points per thread in registers.
//
// The arithmetic is the contract stated in oracle/tfhe_oracle.c (radix-2 DIF
// forward with W[k] = e^{+2 pi i k / 512}, radix-2 DIT inverse with conj(W),
// cmul(x, w) = (fma(xr, wr, -(xi*wi)), fma(xr, wi, xi*wr))): three radix-2
// stages are fused per register pass, the passes exchange through a swizzled
// shared-memory tile, and every butterfly performs exactly the oracle's
// roundings (all ops are __*_rn intrinsics, so nvcc cannot contract them).
// Multiplications by exactly 1 and by exactly +-i are skipped -- exact, so the
// results stay bit-identical to the oracle.
//
// Register layouts (M = 512, thread t in [0, 64), t = 8k + r):
//   pass 0 : x[q] = position t + 64 q        (natural order: the twisted input)
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
__device__ __forceinline__ double2 cadd(double2 a, double2 b)
{
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b)
{
    return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 mul_i(double2 w) { return make_double2(-w.y, w.x); }
__device__ __forceinline__ double2 conj2(double2 w) { return make_double2(w.x, -w.y); }

// forward DIF butterflies
__device__ __forceinline__ void dif(double2& u, double2& v, double2 w)
{
    const double2 d = csub(u, v);
    u = cadd(u, v);
    v = cmul(d, w);
}
__device__ __forceinline__ void dif_1(double2& u, double2& v)
{
    const double2 d = csub(u, v);
    u = cadd(u, v);
    v = d;
}
__device__ __forceinline__ void dif_i(double2& u, double2& v)
{
    const double2 d = csub(u, v);
    u = cadd(u, v);
    v = mul_i(d);
}
// inverse DIT butterflies (wc = conj(W) already applied by the caller)
__device__ __forceinline__ void dit(double2& u, double2& v, double2 wc)
{
    const double2 tt = cmul(v, wc);
    v = csub(u, tt);
    u = cadd(u, tt);
}
__device__ __forceinline__ void dit_1(double2& u, double2& v)
{
    const double2 tt = v;
    v = csub(u, tt);
    u = cadd(u, tt);
}
__device__ __forceinline__ void dit_mi(double2& u, double2& v)  // conj(i) = -i
{
    const double2 tt = make_double2(v.y, -v.x);
    v = csub(u, tt);
    u = cadd(u, tt);
}

// Exchange tile layout: position 64k + 8m + r (k, m, r in [0, 8)) lives at slot
// 72k + 9m + r (576 slots).  Every register layout then addresses its 8 elements as
// base + constant (72 q, 9 m or r), and each quarter warp (8 lanes x 16 B) hits 8
// distinct 16-byte bank groups in all three layouts: conflict-free.
constexpr int XTILE = 576;
__device__ __forceinline__ int slot_of(int k, int m, int r) { return 72 * k + 9 * m + r; }

// Per-thread twiddles, constant for the whole kernel.
struct Twiddles {
    double2 p0a, p0b, p0c, p0d;  // W[t], W[t+64], W[2t], W[4t]
    double2 p1a, p1b, p1c, p1d;  // W[8r], W[8r+64], W[16r], W[32r]
    double2 w64;                 // W[64]
};

__device__ __forceinline__ Twiddles load_twiddles(const double2* __restrict__ W, int t)
{
    Twiddles tw;
    const int r = t & 7;
    tw.p0a = W[t];
    tw.p0b = W[t + 64];
    tw.p0c = W[2 * t];
    tw.p0d = W[4 * t];
    tw.p1a = W[8 * r];
    tw.p1b = W[8 * r + 64];
    tw.p1c = W[16 * r];
    tw.p1d = W[32 * r];
    tw.w64 = W[64];
    return tw;
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
template <class Bar>
__device__ __forceinline__ void exch_p2_to_p1(double2 x[8], double2* buf, int t, Bar bar)
{
    bar();  // the warp's previous reads of this single tile are done
    double2* w = buf + slot_of(t >> 3, t & 7, 0);
#pragma unroll
    for (int q = 0; q < 8; q++)
        w[q] = x[q];
    bar();
    const double2* rd = buf + slot_of(t >> 3, 0, t & 7);
#pragma unroll
    for (int m = 0; m < 8; m++)
        x[m] = rd[9 * m];
}
template <class Bar>
__device__ __forceinline__ void exch_p1_to_p0(double2 x[8], double2* buf, int t, Bar bar)
{
    double2* w = buf + slot_of(t >> 3, 0, t & 7);
#pragma unroll
    for (int m = 0; m < 8; m++)
        w[9 * m] = x[m];
    bar();
    const double2* rd = buf + slot_of(0, t >> 3, t & 7);
#pragma unroll
    for (int q = 0; q < 8; q++)
        x[q] = rd[72 * q];
}

// Forward transform of the twisted input x (pass-0 layout) -> frequency slots
// (pass-2 layout).  bufs: two 512-entry double2 tiles (double buffering).
// bufX: cross-warp exchange tile (needs the 64-thread barrier `bar`);
// bufW: intra-warp exchange tile (after DIF stage 0 the two 256-point halves are
// independent and warp w owns half w in passes 1 and 2, so `wbar` = __syncwarp).
template <class Bar, class WBar>
__device__ __forceinline__ void fft_forward(double2 x[8], const Twiddles& tw, double2* buf0,
                                            double2* buf1, int t, Bar bar, WBar wbar)
{
    // pass 0: stages 0, 1, 2 (h = 256, 128, 64)
    dif(x[0], x[4], tw.p0a);
    dif(x[1], x[5], tw.p0b);
    dif(x[2], x[6], mul_i(tw.p0a));
    dif(x[3], x[7], mul_i(tw.p0b));
    dif(x[0], x[2], tw.p0c);
    dif(x[1], x[3], mul_i(tw.p0c));
    dif(x[4], x[6], tw.p0c);
    dif(x[5], x[7], mul_i(tw.p0c));
    dif(x[0], x[1], tw.p0d);
    dif(x[2], x[3], tw.p0d);
    dif(x[4], x[5], tw.p0d);
    dif(x[6], x[7], tw.p0d);
    exch_p0_to_p1(x, buf0, t, bar);
    // pass 1: stages 3, 4, 5 (h = 32, 16, 8)
    dif(x[0], x[4], tw.p1a);
    dif(x[1], x[5], tw.p1b);
    dif(x[2], x[6], mul_i(tw.p1a));
    dif(x[3], x[7], mul_i(tw.p1b));
    dif(x[0], x[2], tw.p1c);
    dif(x[1], x[3], mul_i(tw.p1c));
    dif(x[4], x[6], tw.p1c);
    dif(x[5], x[7], mul_i(tw.p1c));
    dif(x[0], x[1], tw.p1d);
    dif(x[2], x[3], tw.p1d);
    dif(x[4], x[5], tw.p1d);
    dif(x[6], x[7], tw.p1d);
    exch_p1_to_p2(x, buf1, t, wbar);
    // pass 2: stages 6, 7, 8 (h = 4, 2, 1) -- twiddles W[64 q], W[128 (q&1)], W[0]
    dif_1(x[0], x[4]);
    dif(x[1], x[5], tw.w64);
    dif_i(x[2], x[6]);
    dif(x[3], x[7], mul_i(tw.w64));
    dif_1(x[0], x[2]);
    dif_i(x[1], x[3]);
    dif_1(x[4], x[6]);
    dif_i(x[5], x[7]);
    dif_1(x[0], x[1]);
    dif_1(x[2], x[3]);
    dif_1(x[4], x[5]);
    dif_1(x[6], x[7]);
}

// Inverse transform (unscaled) of frequency slots (pass-2 layout) -> natural order
// (pass-0 layout).  The 1/M scale lives in the untwist table.
template <class Bar, class WBar>
__device__ __forceinline__ void fft_inverse(double2 x[8], const Twiddles& tw, double2* buf0,
                                            double2* buf1, int t, Bar bar, WBar wbar)
{
    // pass 2^-1: stages 8, 7, 6
    dit_1(x[0], x[1]);
    dit_1(x[2], x[3]);
    dit_1(x[4], x[5]);
    dit_1(x[6], x[7]);
    dit_1(x[0], x[2]);
    dit_mi(x[1], x[3]);
    dit_1(x[4], x[6]);
    dit_mi(x[5], x[7]);
    dit_1(x[0], x[4]);
    dit(x[1], x[5], conj2(tw.w64));
    dit_mi(x[2], x[6]);
    dit(x[3], x[7], conj2(mul_i(tw.w64)));
    exch_p2_to_p1(x, buf1, t, wbar);
    // pass 1^-1: stages 5, 4, 3
    dit(x[0], x[1], conj2(tw.p1d));
    dit(x[2], x[3], conj2(tw.p1d));
    dit(x[4], x[5], conj2(tw.p1d));
    dit(x[6], x[7], conj2(tw.p1d));
    dit(x[0], x[2], conj2(tw.p1c));
    dit(x[1], x[3], conj2(mul_i(tw.p1c)));
    dit(x[4], x[6], conj2(tw.p1c));
    dit(x[5], x[7], conj2(mul_i(tw.p1c)));
    dit(x[0], x[4], conj2(tw.p1a));
    dit(x[1], x[5], conj2(tw.p1b));
    dit(x[2], x[6], conj2(mul_i(tw.p1a)));
    dit(x[3], x[7], conj2(mul_i(tw.p1b)));
    exch_p1_to_p0(x, buf0, t, bar);
    // pass 0^-1: stages 2, 1, 0
    dit(x[0], x[1], conj2(tw.p0d));
    dit(x[2], x[3], conj2(tw.p0d));
    dit(x[4], x[5], conj2(tw.p0d));
    dit(x[6], x[7], conj2(tw.p0d));
    dit(x[0], x[2], conj2(tw.p0c));
    dit(x[1], x[3], conj2(mul_i(tw.p0c)));
    dit(x[4], x[6], conj2(tw.p0c));
    dit(x[5], x[7], conj2(mul_i(tw.p0c)));
    dit(x[0], x[4], conj2(tw.p0a));
    dit(x[1], x[5], conj2(tw.p0b));
    dit(x[2], x[6], conj2(mul_i(tw.p0a)));
    dit(x[3], x[7], conj2(mul_i(tw.p0b)));
}

// ---- paired transforms: two independent polynomials per thread in lockstep; they share
// every exchange barrier and the compiler interleaves their butterflies (2x ILP).  The
// per-polynomial arithmetic is exactly fft_forward / fft_inverse.
__device__ __forceinline__ void pass0_fwd(double2 x[8], const Twiddles& tw)
{
    dif(x[0], x[4], tw.p0a);
    dif(x[1], x[5], tw.p0b);
    dif(x[2], x[6], mul_i(tw.p0a));
    dif(x[3], x[7], mul_i(tw.p0b));
    dif(x[0], x[2], tw.p0c);
    dif(x[1], x[3], mul_i(tw.p0c));
    dif(x[4], x[6], tw.p0c);
    dif(x[5], x[7], mul_i(tw.p0c));
    dif(x[0], x[1], tw.p0d);
    dif(x[2], x[3], tw.p0d);
    dif(x[4], x[5], tw.p0d);
    dif(x[6], x[7], tw.p0d);
}
__device__ __forceinline__ void pass1_fwd(double2 x[8], const Twiddles& tw)
{
    dif(x[0], x[4], tw.p1a);
    dif(x[1], x[5], tw.p1b);
    dif(x[2], x[6], mul_i(tw.p1a));
    dif(x[3], x[7], mul_i(tw.p1b));
    dif(x[0], x[2], tw.p1c);
    dif(x[1], x[3], mul_i(tw.p1c));
    dif(x[4], x[6], tw.p1c);
    dif(x[5], x[7], mul_i(tw.p1c));
    dif(x[0], x[1], tw.p1d);
    dif(x[2], x[3], tw.p1d);
    dif(x[4], x[5], tw.p1d);
    dif(x[6], x[7], tw.p1d);
}
__device__ __forceinline__ void pass2_fwd(double2 x[8], const Twiddles& tw)
{
    dif_1(x[0], x[4]);
    dif(x[1], x[5], tw.w64);
    dif_i(x[2], x[6]);
    dif(x[3], x[7], mul_i(tw.w64));
    dif_1(x[0], x[2]);
    dif_i(x[1], x[3]);
    dif_1(x[4], x[6]);
    dif_i(x[5], x[7]);
    dif_1(x[0], x[1]);
    dif_1(x[2], x[3]);
    dif_1(x[4], x[5]);
    dif_1(x[6], x[7]);
}
__device__ __forceinline__ void pass2_inv(double2 x[8], const Twiddles& tw)
{
    dit_1(x[0], x[1]);
    dit_1(x[2], x[3]);
    dit_1(x[4], x[5]);
    dit_1(x[6], x[7]);
    dit_1(x[0], x[2]);
    dit_mi(x[1], x[3]);
    dit_1(x[4], x[6]);
    dit_mi(x[5], x[7]);
    dit_1(x[0], x[4]);
    dit(x[1], x[5], conj2(tw.w64));
    dit_mi(x[2], x[6]);
    dit(x[3], x[7], conj2(mul_i(tw.w64)));
}
__device__ __forceinline__ void pass1_inv(double2 x[8], const Twiddles& tw)
{
    dit(x[0], x[1], conj2(tw.p1d));
    dit(x[2], x[3], conj2(tw.p1d));
    dit(x[4], x[5], conj2(tw.p1d));
    dit(x[6], x[7], conj2(tw.p1d));
    dit(x[0], x[2], conj2(tw.p1c));
    dit(x[1], x[3], conj2(mul_i(tw.p1c)));
    dit(x[4], x[6], conj2(tw.p1c));
    dit(x[5], x[7], conj2(mul_i(tw.p1c)));
    dit(x[0], x[4], conj2(tw.p1a));
    dit(x[1], x[5], conj2(tw.p1b));
    dit(x[2], x[6], conj2(mul_i(tw.p1a)));
    dit(x[3], x[7], conj2(mul_i(tw.p1b)));
}
__device__ __forceinline__ void pass0_inv(double2 x[8], const Twiddles& tw)
{
    dit(x[0], x[1], conj2(tw.p0d));
    dit(x[2], x[3], conj2(tw.p0d));
    dit(x[4], x[5], conj2(tw.p0d));
    dit(x[6], x[7], conj2(tw.p0d));
    dit(x[0], x[2], conj2(tw.p0c));
    dit(x[1], x[3], conj2(mul_i(tw.p0c)));
    dit(x[4], x[6], conj2(tw.p0c));
    dit(x[5], x[7], conj2(mul_i(tw.p0c)));
    dit(x[0], x[4], conj2(tw.p0a));
    dit(x[1], x[5], conj2(tw.p0b));
    dit(x[2], x[6], conj2(mul_i(tw.p0a)));
    dit(x[3], x[7], conj2(mul_i(tw.p0b)));
}

// cross tiles c0/c1 are single-buffered: the leading barrier orders this write after
// every thread's previous read of the same tile.
template <class Bar, class WBar>
__device__ __forceinline__ void fft_forward2(double2 x0[8], double2 x1[8], const Twiddles& tw,
                                             double2* c0, double2* c1, double2* w0, double2* w1,
                                             int t, Bar bar, WBar wbar)
{
    pass0_fwd(x0, tw);
    pass0_fwd(x1, tw);
    bar();
    {
        double2* a = c0 + slot_of(0, t >> 3, t & 7);
        double2* b = c1 + slot_of(0, t >> 3, t & 7);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            a[72 * q] = x0[q];
            b[72 * q] = x1[q];
        }
        bar();
        const double2* ra = c0 + slot_of(t >> 3, 0, t & 7);
        const double2* rb = c1 + slot_of(t >> 3, 0, t & 7);
#pragma unroll
        for (int m = 0; m < 8; m++) {
            x0[m] = ra[9 * m];
            x1[m] = rb[9 * m];
        }
    }
    pass1_fwd(x0, tw);
    pass1_fwd(x1, tw);
    {
        wbar();
        double2* a = w0 + slot_of(t >> 3, 0, t & 7);
        double2* b = w1 + slot_of(t >> 3, 0, t & 7);
#pragma unroll
        for (int m = 0; m < 8; m++) {
            a[9 * m] = x0[m];
            b[9 * m] = x1[m];
        }
        wbar();
        const double2* ra = w0 + slot_of(t >> 3, t & 7, 0);
        const double2* rb = w1 + slot_of(t >> 3, t & 7, 0);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            x0[q] = ra[q];
            x1[q] = rb[q];
        }
    }
    pass2_fwd(x0, tw);
    pass2_fwd(x1, tw);
}

template <class Bar, class WBar>
__device__ __forceinline__ void fft_inverse2(double2 x0[8], double2 x1[8], const Twiddles& tw,
                                             double2* c0, double2* c1, double2* w0, double2* w1,
                                             int t, Bar bar, WBar wbar)
{
    pass2_inv(x0, tw);
    pass2_inv(x1, tw);
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
    pass1_inv(x0, tw);
    pass1_inv(x1, tw);
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
    pass0_inv(x0, tw);
    pass0_inv(x1, tw);
}

}  // namespace lpb
