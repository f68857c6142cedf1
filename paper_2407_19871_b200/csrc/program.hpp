// program.hpp -- the circuit scheduler (host C++, no CUDA).
//
// The reference evaluates gates one at a time in program order, each ending in a
// refresh (GateEngine::refresh_gate, gate_engine.hpp:322-328), and parallelises
// only across regions with CPU threads (circuits.hpp:296-321).  Here a gate
// program is lowered to micro-ops and every micro-op is assigned to the earliest
// depth level ("wave") its inputs allow:
//   * AND/OR/XOR/XNOR/NAND/NOR : one blind rotation (BR) + one key switch (KS)
//   * MUX(s, a, b)             : BR(-1/8 + s + a), BR(-1/8 - s + b), then one KS of
//                                their N-dim sum + 1/8 (TFHE bootsMUX).  The two
//                                halves are scheduled independently, so in the
//                                comparator chain t0 = MUX(t1, t0, b_i)
//                                (circuits.hpp:202-207) the "else" half leaves the
//                                critical path.
//   * NOT/COPY/CONST           : free linear ops, run at the start of a wave.
// A wave is launched as: linear kernel, one batched BR kernel, one batched KS
// kernel.  N-dim intermediates live in a scratch pool recycled across waves.
#pragma once
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/locpir_b200.h"
#include "kernels.cuh"

namespace lpb {

struct Plan {
    std::vector<std::vector<BrItem>> br;    // per wave
    std::vector<std::vector<KsItem>> ks;    // per wave
    std::vector<std::vector<LinItem>> lin;  // per wave (run before the wave's BR)
    uint32_t scratch = 0;                   // N-dim scratch slots needed
    uint64_t n_br = 0, n_ks = 0;
    uint64_t counts[10] = {0};              // and or xor xnor not mux nand nor units, [9] flagged 3-input gates (MAJ, XOR3)
    uint32_t waves() const { return (uint32_t)br.size(); }
};

struct GateForm {
    uint32_t off;
    int32_t c0, c1;
};

// Linear forms of the bootstrapped gates (gate_engine.hpp:196-240, plus NAND/NOR).
inline bool gate_form(uint32_t kind, GateForm& f)
{
    switch (kind) {
    case LOCPIR_B200_AND: f = {0xE0000000u, 1, 1}; return true;
    case LOCPIR_B200_OR: f = {0x20000000u, 1, 1}; return true;
    case LOCPIR_B200_XOR: f = {0x40000000u, 2, 2}; return true;
    case LOCPIR_B200_XNOR: f = {0xC0000000u, -2, -2}; return true;
    case LOCPIR_B200_NAND: f = {0x20000000u, -1, -1}; return true;
    case LOCPIR_B200_NOR: f = {0xE0000000u, -1, -1}; return true;
    case LOCPIR_B200_ANDNY: f = {0xE0000000u, -1, 1}; return true;
    case LOCPIR_B200_ORNY: f = {0x20000000u, -1, 1}; return true;
    default: return false;
    }
}

// Per-slot scheduling state: ready waves for BR / linear use and read/write flags.
struct SlotInfo {
    uint32_t rbr = 0, rlin = 0;
    uint8_t written = 0, read = 0;
};

// Dense table when slot ids are proportional to the program size (pool layouts always
// are), hash map otherwise -- planning 65,536 gates drops from ~35 ms to ~2 ms.
class SlotTable {
  public:
    SlotTable(const locpir_b200_gate_op* ops, uint64_t count)
    {
        uint64_t mx = 0;
        for (uint64_t g = 0; g < count; g++)
            for (uint32_t s : {ops[g].in0, ops[g].in1, ops[g].in2, ops[g].out})
                if (s != SLOT_NONE && s > mx)
                    mx = s;
        if (mx < 8 * count + (1u << 16))
            dense_.resize(mx + 1);
    }
    SlotInfo& operator[](uint32_t s) { return dense_.empty() ? sparse_[s] : dense_[s]; }
    uint32_t rbr(uint32_t s) const { return find(s).rbr; }
    uint32_t rlin(uint32_t s) const { return find(s).rlin; }

  private:
    const SlotInfo& find(uint32_t s) const
    {
        static const SlotInfo none;
        if (!dense_.empty())
            return dense_[s];
        auto it = sparse_.find(s);
        return it == sparse_.end() ? none : it->second;
    }
    std::vector<SlotInfo> dense_;
    std::unordered_map<uint32_t, SlotInfo> sparse_;
};

inline Plan build_plan(const locpir_b200_gate_op* ops, uint64_t count)
{
    Plan P;
    SlotTable st(ops, count);
    struct Tmp {
        uint32_t wave_br;
        uint32_t wave_ks = 0;
    };
    std::vector<Tmp> tmps;
    tmps.reserve(count);
    // temporary ids (N-dim values) referenced by BR out / KS in until slots are assigned
    auto ready_br = [&](uint32_t s) { return st.rbr(s); };
    auto ready_lin = [&](uint32_t s) { return st.rlin(s); };
    auto ensure = [&](uint32_t w) {
        if (P.br.size() <= w) {
            P.br.resize(w + 1);
            P.ks.resize(w + 1);
            P.lin.resize(w + 1);
        }
    };
    auto use = [&](uint32_t s) {
        if (s == SLOT_NONE)
            throw std::invalid_argument("gate operand slot missing");
        st[s].read = 1;
    };
    auto def = [&](uint32_t s) {
        if (s == SLOT_NONE)
            throw std::invalid_argument("gate output slot missing");
        SlotInfo& si = st[s];
        if (si.written)
            throw std::invalid_argument("slot " + std::to_string(s) +
                                        " written twice in one program");
        if (si.read)
            throw std::invalid_argument("slot " + std::to_string(s) +
                                        " written after being read in the same program");
        si.written = 1;
    };
    auto new_br = [&](uint32_t w, uint32_t in0, uint32_t in1, int32_t c0, int32_t c1,
                      uint32_t off, uint32_t in2 = SLOT_NONE, int32_t c2 = 0) {
        ensure(w);
        const uint32_t id = (uint32_t)tmps.size();
        tmps.push_back({w});
        P.br[w].push_back({in0, in1, c0, c1, off, id, in2, c2});
        P.n_br++;
        return id;
    };

    for (uint64_t g = 0; g < count; g++) {
        const locpir_b200_gate_op& op = ops[g];
        GateForm f;
        if (gate_form(op.kind, f)) {
            use(op.in0);
            use(op.in1);
            def(op.out);
            const uint32_t w = std::max(ready_br(op.in0), ready_br(op.in1));
            const uint32_t id = new_br(w, op.in0, op.in1, f.c0, f.c1, f.off);
            P.ks[w].push_back({id, SLOT_NONE, 0u, op.out});
            tmps[id].wave_ks = w;
            P.n_ks++;
            st[op.out].rbr = st[op.out].rlin = w + 1;
            // counters: ANDNY / ORNY count as AND / OR
            static const int cidx[] = {0, 1, 2, 3, 6, -1, -1, 7, -1, -1, 0, 1};
            P.counts[cidx[op.kind]]++;
        } else if (op.kind == LOCPIR_B200_MAJ || op.kind == LOCPIR_B200_XOR3) {
            // 3-input majority: BS(in0 + in1 + in2) -- the sum of three +-1/8 never hits 0;
            // 3-input XOR: BS(-2 (in0 + in1 + in2)) -- +1/4 for an odd count, -1/4 for even
            use(op.in0);
            use(op.in1);
            use(op.in2);
            def(op.out);
            const uint32_t w =
                std::max(std::max(ready_br(op.in0), ready_br(op.in1)), ready_br(op.in2));
            const int32_t k = op.kind == LOCPIR_B200_MAJ ? 1 : -2;
            const uint32_t id = new_br(w, op.in0, op.in1, k, k, 0u, op.in2, k);
            P.ks[w].push_back({id, SLOT_NONE, 0u, op.out});
            tmps[id].wave_ks = w;
            P.n_ks++;
            st[op.out].rbr = st[op.out].rlin = w + 1;
            P.counts[9]++;
        } else if (op.kind == LOCPIR_B200_MUX) {
            use(op.in0);
            use(op.in1);
            use(op.in2);
            def(op.out);
            const uint32_t w1 = std::max(ready_br(op.in0), ready_br(op.in1));
            const uint32_t w2 = std::max(ready_br(op.in0), ready_br(op.in2));
            const uint32_t t1 = new_br(w1, op.in0, op.in1, 1, 1, 0xE0000000u);
            const uint32_t t2 = new_br(w2, op.in0, op.in2, -1, 1, 0xE0000000u);
            const uint32_t w = std::max(w1, w2);
            ensure(w);
            P.ks[w].push_back({t1, t2, 0x20000000u, op.out});
            tmps[t1].wave_ks = tmps[t2].wave_ks = w;
            P.n_ks++;
            st[op.out].rbr = st[op.out].rlin = w + 1;
            P.counts[5]++;
        } else if (op.kind == LOCPIR_B200_NOT || op.kind == LOCPIR_B200_COPY) {
            use(op.in0);
            def(op.out);
            const uint32_t w = ready_lin(op.in0);
            ensure(w);
            P.lin[w].push_back({op.kind == LOCPIR_B200_NOT ? 0u : 1u, op.in0, op.out, 0});
            st[op.out].rbr = w;
            st[op.out].rlin = w + 1;
            if (op.kind == LOCPIR_B200_NOT)
                P.counts[4]++;
        } else if (op.kind == LOCPIR_B200_CONST) {
            def(op.out);
            ensure(0);
            P.lin[0].push_back({2u, op.in0 ? 0x20000000u : 0xE0000000u, op.out, 0});
            st[op.out].rbr = 0;
            st[op.out].rlin = 1;
        } else {
            throw std::invalid_argument("unknown gate kind " + std::to_string(op.kind));
        }
    }
    P.counts[8] = P.counts[0] + P.counts[1] + P.counts[2] + P.counts[3] + P.counts[6] +
                  P.counts[7] + 2 * P.counts[5] + P.counts[9];

    // assign N-dim scratch slots: a value lives from its BR wave to its KS wave
    std::vector<uint32_t> phys(tmps.size(), SLOT_NONE), freelist;
    uint32_t next = 0;
    for (uint32_t w = 0; w < P.br.size(); w++) {
        for (BrItem& b : P.br[w]) {
            uint32_t s;
            if (!freelist.empty()) {
                s = freelist.back();
                freelist.pop_back();
            } else {
                s = next++;
            }
            phys[b.out] = s;
            b.out = s;
        }
        for (KsItem& k : P.ks[w]) {
            k.in0 = phys[k.in0];
            freelist.push_back(k.in0);
            if (k.in1 != SLOT_NONE) {
                k.in1 = phys[k.in1];
                freelist.push_back(k.in1);
            }
        }
    }
    P.scratch = next;
    return P;
}

}  // namespace lpb
