// circuits.hpp -- LocPIR circuits emitted as gate programs (host C++, no CUDA).
//
// Gate-for-gate restatement of the reference circuits (circuits.hpp:187-324) over
// pool slots, so gate counts are exactly N(12l + 2m + 3) units per query
// (bench.hpp:35-43).  The scheduler (program.hpp) batches every independent gate
// of all queries and regions into one level.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/locpir_b200.h"

namespace lpb {

struct Emitter {
    std::vector<locpir_b200_gate_op>* ops;
    uint64_t next;  // next free scratch slot
    uint32_t fresh() { return (uint32_t)next++; }
    uint32_t gate(uint32_t kind, uint32_t a, uint32_t b = 0xFFFFFFFFu, uint32_t c = 0xFFFFFFFFu,
                  uint32_t out = 0xFFFFFFFFu)
    {
        if (out == 0xFFFFFFFFu)
            out = fresh();
        ops->push_back({kind, a, b, c, out});
        return out;
    }
};

// hom_less (circuits.hpp:191-209): flip both sign bits (free NOTs), then
// t0 = 0; t1 = XNOR(a_i, b_i); t0 = MUX(t1, t0, b_i) for i = 0..l-1.
inline uint32_t emit_less(Emitter& e, const uint32_t* a, const uint32_t* b, uint32_t l)
{
    const uint32_t a_sign = e.gate(LOCPIR_B200_NOT, a[l - 1]);
    const uint32_t b_sign = e.gate(LOCPIR_B200_NOT, b[l - 1]);
    uint32_t t0 = e.gate(LOCPIR_B200_CONST, 0);
    for (uint32_t i = 0; i < l; i++) {
        const uint32_t ai = (i + 1 == l) ? a_sign : a[i];
        const uint32_t bi = (i + 1 == l) ? b_sign : b[i];
        const uint32_t t1 = e.gate(LOCPIR_B200_XNOR, ai, bi);
        t0 = e.gate(LOCPIR_B200_MUX, t1, t0, bi);
    }
    return t0;
}

// Flagged comparator (majority borrow chain): with both sign bits flipped (free NOTs),
// a < b (signed) = borrow out of a' - b'; borrow_{i+1} = MAJ(NOT a'_i, b'_i, borrow_i)
// with borrow_0 = Enc(0) trivial.  One bootstrap per bit.  NOT a'_{l-1} = a_{l-1}.
inline uint32_t emit_less_maj(Emitter& e, const uint32_t* a, const uint32_t* b, uint32_t l)
{
    uint32_t borrow = e.gate(LOCPIR_B200_CONST, 0);
    for (uint32_t i = 0; i < l; i++) {
        const bool sign = i + 1 == l;
        const uint32_t na = sign ? a[i] : e.gate(LOCPIR_B200_NOT, a[i]);
        const uint32_t bi = sign ? e.gate(LOCPIR_B200_NOT, b[i]) : b[i];
        borrow = e.gate(LOCPIR_B200_MAJ, na, bi, borrow);
    }
    return borrow;
}

// ---- flagged latency mode: log-depth (tree) comparator ------------------------------
// Same function as hom_less.  With both sign bits flipped, per bit
//   lt_i = NOT a'_i AND b'_i,  eq_i = (a'_i == b'_i)
// and pairs merge up a balanced tree (hi = the more significant half):
//   lt = eq_hi ? lt_lo : lt_hi   (MUX; lt_hi and eq_hi are exclusive)
//   eq = eq_hi AND eq_lo
// Depth log2(l) (+1 with an encrypted b) instead of l, for latency-bound batches (cfg1).
// b bits may be plaintext constants (folded) or pool slots; constants propagate for free.
struct TBit {
    bool is_const;
    int v;
    uint32_t slot;
    static TBit c(int x) { return {true, x ? 1 : 0, 0}; }
    static TBit s(uint32_t x) { return {false, 0, x}; }
};

struct TreeOps {
    Emitter& e;
    uint32_t mat(TBit x) { return x.is_const ? e.gate(LOCPIR_B200_CONST, (uint32_t)x.v) : x.slot; }
    TBit not_(TBit x) { return x.is_const ? TBit::c(!x.v) : TBit::s(e.gate(LOCPIR_B200_NOT, x.slot)); }
    TBit and_(TBit x, TBit y)
    {
        if ((x.is_const && !x.v) || (y.is_const && !y.v))
            return TBit::c(0);
        if (x.is_const)
            return y;
        if (y.is_const)
            return x;
        return TBit::s(e.gate(LOCPIR_B200_AND, x.slot, y.slot));
    }
    TBit mux(TBit s_, TBit a, TBit b)  // s ? a : b
    {
        if (s_.is_const)
            return s_.v ? a : b;
        if (a.is_const && b.is_const)
            return a.v == b.v ? a : (a.v ? s_ : not_(s_));
        if (a.is_const)  // s ? 1 : b = s OR b ; s ? 0 : b = NOT s AND b
            return TBit::s(e.gate(a.v ? LOCPIR_B200_OR : LOCPIR_B200_ANDNY, s_.slot, b.slot));
        if (b.is_const)  // s ? a : 1 = NOT s OR a ; s ? a : 0 = s AND a
            return TBit::s(e.gate(b.v ? LOCPIR_B200_ORNY : LOCPIR_B200_AND, s_.slot, a.slot));
        return TBit::s(e.gate(LOCPIR_B200_MUX, s_.slot, a.slot, b.slot));
    }
};

// a: l slots; b: l TBits (constants or slots).  Returns the slot of a < b (signed).
inline uint32_t emit_less_tree(Emitter& e, const uint32_t* a, const TBit* b, uint32_t l)
{
    TreeOps t{e};
    std::vector<TBit> lt(l), eq(l);
    for (uint32_t i = 0; i < l; i++) {
        const bool sign = i + 1 == l;
        TBit ai = TBit::s(a[i]);
        TBit bi = b[i];
        // a'_i = NOT a_{l-1} at the sign position (free); NOT a'_i is then a_{l-1}
        const TBit na = sign ? ai : t.not_(ai);
        const TBit ap = sign ? t.not_(ai) : ai;
        if (sign)
            bi = t.not_(bi);
        if (bi.is_const) {
            lt[i] = bi.v ? na : TBit::c(0);
            eq[i] = bi.v ? ap : na;
        } else {
            lt[i] = TBit::s(e.gate(LOCPIR_B200_ANDNY, t.mat(ap), bi.slot));
            eq[i] = TBit::s(e.gate(LOCPIR_B200_XNOR, t.mat(ap), bi.slot));
        }
    }
    // merge [lo, hi) ranges bottom-up; level vectors hold (lt, eq) of consecutive groups
    while (lt.size() > 1) {
        std::vector<TBit> nlt, neq;
        for (size_t i = 0; i + 1 < lt.size(); i += 2) {
            nlt.push_back(t.mux(eq[i + 1], lt[i], lt[i + 1]));
            neq.push_back(lt.size() == 2 ? TBit::c(0) : t.and_(eq[i + 1], eq[i]));
        }
        if (lt.size() & 1) {
            nlt.push_back(lt.back());
            neq.push_back(eq.back());
        }
        lt.swap(nlt);
        eq.swap(neq);
    }
    return t.mat(lt[0]);
}

// hom_less_equal (circuits.hpp:212-216): NOT(b < a).
inline uint32_t emit_less_equal(Emitter& e, const uint32_t* a, const uint32_t* b, uint32_t l)
{
    return e.gate(LOCPIR_B200_NOT, emit_less(e, b, a, l));
}

inline uint64_t loc_pir_scratch(uint32_t Q, uint32_t R, uint32_t l, uint32_t m)
{
    // per region: 4 comparators x (at most 7l + 4 slots: the reference chain needs
    // 2 NOT + 1 CONST + 2l, the majority chain 2l + 1, the tree 5l) + 2 NOT + 3 AND +
    // m AND; per query and bit column: 1 CONST + (R - 1) XOR
    const uint64_t per_region = 4ull * (4 + 7ull * l) + 2 + 3 + m;
    const uint64_t per_query = (uint64_t)R * per_region + (uint64_t)m * (1 + R);
    return (uint64_t)Q * per_query;
}

// Balanced XOR tree over one bit column.  mode 1: root XOR Enc(0) -> dst (N XOR units for
// N boxes, as the reference chain).  mode 2 (box-sharded partial): the root
// is copied to dst without the XOR with Enc(0) (N-1 units); the rank-0 combine adds one
// XOR per shard plus the one with Enc(0), so the total stays N units.
// ternary (flagged modes): XOR3 nodes (one bootstrap each), so the tree has ceil(log3 N)
// levels and about (N - 1) / 2 bootstraps instead of log2 N levels and N - 1.
inline void emit_xor_root(Emitter& e, std::vector<uint32_t> lvl, uint32_t zero, uint32_t dst,
                          int mode, bool ternary = false)
{
    while (lvl.size() > 1) {
        std::vector<uint32_t> nxt;
        size_t i = 0;
        if (ternary)
            for (; i + 2 < lvl.size(); i += 3)
                nxt.push_back(e.gate(LOCPIR_B200_XOR3, lvl[i], lvl[i + 1], lvl[i + 2]));
        for (; i + 1 < lvl.size(); i += 2)
            nxt.push_back(e.gate(LOCPIR_B200_XOR, lvl[i], lvl[i + 1]));
        if (i < lvl.size())
            nxt.push_back(lvl.back());
        lvl.swap(nxt);
    }
    if (mode == 2 || zero == 0xFFFFFFFFu)
        e.gate(LOCPIR_B200_COPY, lvl[0], 0xFFFFFFFFu, 0xFFFFFFFFu, dst);
    else
        e.gate(LOCPIR_B200_XOR, zero, lvl[0], 0xFFFFFFFFu, dst);
}

// XOR-sum of one bit column into dst.  The reference starts every column from Enc(0)
// (circuits.hpp:257-261) and bootstraps that XOR too; the flagged modes (already not the
// reference gate count) skip it -- the XOR with a trivial zero only refreshes a value that
// is itself a fresh bootstrap output, and it costs a whole circuit level (the last one) --
// and reduce the column with a ternary XOR3 tree.
inline void emit_xor_column(Emitter& e, const std::vector<uint32_t>& lvl, uint32_t dst,
                            int xor_tree, bool flagged)
{
    const uint32_t zero = flagged && xor_tree != 2 ? 0xFFFFFFFFu : e.gate(LOCPIR_B200_CONST, 0);
    if (xor_tree) {
        emit_xor_root(e, lvl, zero, dst, xor_tree, flagged);
        return;
    }
    const size_t R = lvl.size();
    uint32_t acc = zero;
    for (size_t r = 0; r < R; r++) {
        const uint32_t o = r + 1 == R ? dst : 0xFFFFFFFFu;
        if (acc == 0xFFFFFFFFu)  // flagged chain: starts from the first term
            acc = R == 1 ? e.gate(LOCPIR_B200_COPY, lvl[0], 0xFFFFFFFFu, 0xFFFFFFFFu, o) : lvl[0];
        else
            acc = e.gate(LOCPIR_B200_XOR, acc, lvl[r], 0xFFFFFFFFu, o);
    }
}

// loc_pir (circuits.hpp:276-324) for Q queries.  xor_tree = 0 keeps the
// reference's N-long chain per bit column (circuits.hpp:257-261); 1 uses a
// balanced tree of N-1 XORs plus one XOR with Enc(0): still N*m XOR units.
// svc(q, r, j) -> pool slot of service bit j of region r as seen by query q (shared
// across queries for one session; per session in the cross-session batcher).
template <class SvcFn>
inline void emit_loc_pir_fn(std::vector<locpir_b200_gate_op>& ops, uint32_t Q, uint32_t R,
                            uint32_t l, uint32_t m, const uint32_t* xs, const uint32_t* ys,
                            const uint32_t* bnd, SvcFn svc, const uint32_t* out,
                            uint64_t scratch_first, int xor_tree, int cmp = 0)
{
    // cmp: 0 = reference XNOR/MUX chain, 1 = majority borrow chain, 2 = log-depth tree
    std::vector<TBit> tb(l);
    auto lt = [&](Emitter& e, const uint32_t* a, const uint32_t* b) {
        if (cmp == 1)
            return emit_less_maj(e, a, b, l);
        if (cmp == 2) {
            for (uint32_t i = 0; i < l; i++)
                tb[i] = TBit::s(b[i]);
            return emit_less_tree(e, a, tb.data(), l);
        }
        return emit_less(e, a, b, l);
    };
    auto le = [&](Emitter& e, const uint32_t* a, const uint32_t* b) {  // NOT(b < a)
        return e.gate(LOCPIR_B200_NOT, lt(e, b, a));
    };
    Emitter e{&ops, scratch_first};
    std::vector<uint32_t> masked((size_t)R * m);
    for (uint32_t q = 0; q < Q; q++) {
        const uint32_t* x = xs + (size_t)q * l;
        const uint32_t* y = ys + (size_t)q * l;
        for (uint32_t r = 0; r < R; r++) {
            const uint32_t* x1 = bnd + ((size_t)r * 4 + 0) * l;
            const uint32_t* x2 = bnd + ((size_t)r * 4 + 1) * l;
            const uint32_t* y1 = bnd + ((size_t)r * 4 + 2) * l;
            const uint32_t* y2 = bnd + ((size_t)r * 4 + 3) * l;
            const uint32_t x_l = le(e, x1, x);
            const uint32_t x_r = lt(e, x, x2);
            const uint32_t y_l = le(e, y1, y);
            const uint32_t y_r = lt(e, y, y2);
            const uint32_t v1 = e.gate(LOCPIR_B200_AND, x_l, x_r);
            const uint32_t v2 = e.gate(LOCPIR_B200_AND, y_l, y_r);
            const uint32_t f = e.gate(LOCPIR_B200_AND, v1, v2);
            for (uint32_t j = 0; j < m; j++)  // mask_service (circuits.hpp:219-227)
                masked[(size_t)r * m + j] = e.gate(LOCPIR_B200_AND, f, svc(q, r, j));
        }
        // xor_sum_services (circuits.hpp:240-269); cmp != 0 is a flagged mode
        std::vector<uint32_t> lvl(R);
        for (uint32_t j = 0; j < m; j++) {
            for (uint32_t r = 0; r < R; r++)
                lvl[r] = masked[(size_t)r * m + j];
            emit_xor_column(e, lvl, out[(size_t)q * m + j], xor_tree, cmp != 0);
        }
    }
}

// ---- flagged mode: comparators against a PLAINTEXT word -------------
// Same function as emit_less(a, B) for a known l-bit word B: with the sign bits flipped,
// scan LSB -> MSB keeping t0 = [a' < B'] on the bits seen so far; at bit i
//   b_i = 1 : t0 <- a_i ? t0 : 1 = OR(NOT a_i, t0)
//   b_i = 0 : t0 <- a_i ? 0 : t0 = AND(NOT a_i, t0)
// (XNOR(a_i, b_i) is a free negation or nothing).  While t0 is a known constant the
// update is a free NOT / constant; otherwise one bootstrap (ANDNY / ORNY form).
// Returns the slot of a < B (signed).
struct MaybeConst {
    bool is_const;
    int value;
    uint32_t slot;
};

inline uint32_t emit_less_plain(Emitter& e, const uint32_t* a, int64_t B, uint32_t l)
{
    const uint64_t u = (uint64_t)B;
    MaybeConst t0{true, 0, 0};
    for (uint32_t i = 0; i < l; i++) {
        uint32_t bi = (uint32_t)((u >> i) & 1);
        const bool sign = i + 1 == l;
        if (sign)
            bi ^= 1u;  // b' = NOT b at the sign position; a' = NOT a
        if (t0.is_const) {
            if ((bi == 1 && t0.value == 1) || (bi == 0 && t0.value == 0))
                continue;  // t0 unchanged constant
            // t0 <- NOT a'_i  (a'_i = a_i, or NOT a_{l-1} at the sign bit)
            t0 = {false, 0, sign ? e.gate(LOCPIR_B200_COPY, a[i]) : e.gate(LOCPIR_B200_NOT, a[i])};
            continue;
        }
        if (!sign)
            t0.slot = e.gate(bi ? LOCPIR_B200_ORNY : LOCPIR_B200_ANDNY, a[i], t0.slot);
        else  // NOT a'_{l-1} = a_{l-1}
            t0.slot = e.gate(bi ? LOCPIR_B200_OR : LOCPIR_B200_AND, a[i], t0.slot);
    }
    if (t0.is_const)
        return e.gate(LOCPIR_B200_CONST, (uint32_t)t0.value);
    return t0.slot;
}

inline uint64_t loc_pir_folded_scratch(uint32_t Q, uint32_t R, uint32_t l, uint32_t m)
{
    // per comparator: the folded chain needs l + 2 slots, the folded tree at most 4l + 1
    const uint64_t per_region = 4ull * (4ull * l + 2) + 2 + 3 + m;
    return (uint64_t)Q * ((uint64_t)R * per_region + (uint64_t)m * (1 + R));
}

// loc_pir with plaintext boxes [R][4] = (x1, x2, y1, y2): x1 <= x = NOT(x < x1).
template <class SvcFn>
inline void emit_loc_pir_folded_fn(std::vector<locpir_b200_gate_op>& ops, uint32_t Q, uint32_t R,
                                   uint32_t l, uint32_t m, const uint32_t* xs, const uint32_t* ys,
                                   const int64_t* boxes, SvcFn svc, const uint32_t* out,
                                   uint64_t scratch_first, int xor_tree, bool tree = false)
{
    std::vector<TBit> tb(l);
    auto lt_plain = [&](Emitter& e, const uint32_t* a, int64_t B) {
        if (!tree)
            return emit_less_plain(e, a, B, l);
        for (uint32_t i = 0; i < l; i++)
            tb[i] = TBit::c((int)(((uint64_t)B >> i) & 1));
        return emit_less_tree(e, a, tb.data(), l);
    };
    Emitter e{&ops, scratch_first};
    std::vector<uint32_t> masked((size_t)R * m);
    for (uint32_t q = 0; q < Q; q++) {
        const uint32_t* x = xs + (size_t)q * l;
        const uint32_t* y = ys + (size_t)q * l;
        for (uint32_t r = 0; r < R; r++) {
            const int64_t* bx = boxes + (size_t)r * 4;
            const uint32_t x_l = e.gate(LOCPIR_B200_NOT, lt_plain(e, x, bx[0]));
            const uint32_t x_r = lt_plain(e, x, bx[1]);
            const uint32_t y_l = e.gate(LOCPIR_B200_NOT, lt_plain(e, y, bx[2]));
            const uint32_t y_r = lt_plain(e, y, bx[3]);
            const uint32_t v1 = e.gate(LOCPIR_B200_AND, x_l, x_r);
            const uint32_t v2 = e.gate(LOCPIR_B200_AND, y_l, y_r);
            const uint32_t f = e.gate(LOCPIR_B200_AND, v1, v2);
            for (uint32_t j = 0; j < m; j++)
                masked[(size_t)r * m + j] = e.gate(LOCPIR_B200_AND, f, svc(q, r, j));
        }
        std::vector<uint32_t> lvl(R);
        for (uint32_t j = 0; j < m; j++) {  // flagged mode: no XOR with Enc(0)
            for (uint32_t r = 0; r < R; r++)
                lvl[r] = masked[(size_t)r * m + j];
            emit_xor_column(e, lvl, out[(size_t)q * m + j], xor_tree, true);
        }
    }
}

// Shared service table [R][m] (one session / the reference's single-session server).
inline void emit_loc_pir(std::vector<locpir_b200_gate_op>& ops, uint32_t Q, uint32_t R,
                         uint32_t l, uint32_t m, const uint32_t* xs, const uint32_t* ys,
                         const uint32_t* bnd, const uint32_t* svc, const uint32_t* out,
                         uint64_t scratch_first, int xor_tree, int cmp = 0)
{
    emit_loc_pir_fn(ops, Q, R, l, m, xs, ys, bnd,
                    [&](uint32_t, uint32_t r, uint32_t j) { return svc[(size_t)r * m + j]; }, out,
                    scratch_first, xor_tree, cmp);
}

inline void emit_loc_pir_folded(std::vector<locpir_b200_gate_op>& ops, uint32_t Q, uint32_t R,
                                uint32_t l, uint32_t m, const uint32_t* xs, const uint32_t* ys,
                                const int64_t* boxes, const uint32_t* svc, const uint32_t* out,
                                uint64_t scratch_first, int xor_tree, bool tree = false)
{
    emit_loc_pir_folded_fn(ops, Q, R, l, m, xs, ys, boxes,
                           [&](uint32_t, uint32_t r, uint32_t j) { return svc[(size_t)r * m + j]; },
                           out, scratch_first, xor_tree, tree);
}

}  // namespace lpb
