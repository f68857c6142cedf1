// engine.cu -- device context, ciphertext pool, level-batched execution and the
// C ABI (include/locpir_b200.h).  Host C++ around the sm_100a kernels of
// kernels.cuh; no CPU fallback exists: every gate runs on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/locpir_b200.h"
#include "server.hpp"
#include "circuits.hpp"
#include "kernels.cuh"
#include "ks_tc.cuh"
#include "program.hpp"

using namespace lpb;

namespace {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));              \
    } while (0)

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void reserve(size_t want, cudaStream_t s, bool keep)
    {
        if (want <= n)
            return;
        size_t cap = std::max(want, n + n / 2);
        T* q = nullptr;
        CK(cudaMalloc(&q, cap * sizeof(T)));
        if (keep && p && n)
            CK(cudaMemcpyAsync(q, p, n * sizeof(T), cudaMemcpyDeviceToDevice, s));
        if (p) {
            CK(cudaStreamSynchronize(s));
            CK(cudaFree(p));
        }
        p = q;
        n = cap;
    }
    ~DevBuf()
    {
        if (p)
            cudaFree(p);
    }
};

template <class T>
struct PinnedBuf {
    T* p = nullptr;
    size_t n = 0;
    void reserve(size_t want)
    {
        if (want <= n)
            return;
        if (p)
            cudaFreeHost(p);
        n = std::max(want, n * 2);
        if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) {
            p = nullptr;
            n = 0;
            throw CudaError("cudaMallocHost failed");
        }
    }
    ~PinnedBuf()
    {
        if (p)
            cudaFreeHost(p);
    }
};

struct Timer {
    std::vector<cudaEvent_t> ev[3];  // start/stop pairs per kernel class
    double ms[3] = {0, 0, 0};
    uint64_t launches[3] = {0, 0, 0};
};

}  // namespace

struct locpir_b200_ctx {
    locpir_b200_params p{};
    DevParams dp{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    DevBuf<double2> ftw, itw, TW, bkf;  // per-thread twiddles [8][64] x2, twist [512]
    DevBuf<uint32_t> ksk;
    DevBuf<uint4> kskt;      // KSK in the tiled byte layout of K2t (ks_tc.cuh)
    uint32_t kskt_tiles = 0; // N tiles of 256 byte-columns
    int ks_tc = 1;           // env LOCPIR_B200_KSTC=0: batched levels use K2 instead of K2t
    bool have_keys = false;
    DevBuf<uint32_t> pool_n, pool_N;
    uint64_t pool_slots = 0, scratch_slots = 0;
    DevBuf<BrItem> d_br;
    DevBuf<KsItem> d_ks;
    DevBuf<LinItem> d_lin;
    PinnedBuf<BrItem> h_br;
    PinnedBuf<KsItem> h_ks;
    PinnedBuf<LinItem> h_lin;
    uint64_t counters[9] = {0};
    bool timing = false;
    Timer timer;
    int num_sms = 148;
    // small levels (fewer bootstraps than SMs) take the latency kernels
    int small_levels = 1;
    int use_graphs = 1;   // LOCPIR_B200_GRAPH=0: programs launch without CUDA graphs
    int zero_copy = 1;    // LOCPIR_B200_ZEROCOPY=0: gate_batch_host always copies its inputs
    const uint32_t* ext_a = nullptr;  // zero-copy inputs of the running gate_batch_host
    const uint32_t* ext_b = nullptr;
    uint32_t ext_rows = 0;
    int l2_persist = 1;  // env LOCPIR_B200_L2PERSIST=0 disables
    // env LOCPIR_B200_POISON=<u32>: newly grown pool and scratch memory is filled with this
    // word instead of zeros / left undefined (self-check: results must not depend on it)
    uint32_t poison = 0;
    bool poison_set = false;
    // persisting-L2 window over the frequency-domain BK, attached per K1 launch (never to
    // the caller's stream); the device-wide persisting limit is released by the last
    // context that set it
    bool have_window = false;
    cudaAccessPolicyWindow bk_window{};
    // A batching server on this context owns every pool slot >= server_base; calls from
    // anything else that touch those slots fail (EINVAL) instead of corrupting it.
    uint64_t server_base = UINT64_MAX;
    int server_calls = 0;  // > 0 while a locpir_b200_server_* entry point runs
    DevBuf<uint32_t> ks_partial;
    DevBuf<uint32_t> h2d_stage;  // packed rows for 1-D host copies (k_repack_rows)
    DevBuf<uint32_t> d2h_stage;  // packed rows for 1-D device-to-host copies (k_pack_rows)
};

namespace {

// fill device words with v (pool growth: zeros, or the self-check poison)
void fill_words(locpir_b200_ctx* c, uint32_t* p, size_t words, uint32_t v)
{
    if (!words)
        return;
    if (v == 0) {
        CK(cudaMemsetAsync(p, 0, words * 4, c->stream));
        return;
    }
    k_fill<<<c->num_sms * 4, 256, 0, c->stream>>>(p, words, v);
    CK(cudaGetLastError());
}
// scratch (N-dim) growth: undefined contents, poisoned in self-check runs
void grow_scratch(locpir_b200_ctx* c, uint64_t slots)
{
    const size_t old = c->pool_N.n;
    c->pool_N.reserve((size_t)slots * c->dp.N_stride, c->stream, false);
    if (c->poison_set && c->pool_N.n != old)
        fill_words(c, c->pool_N.p, c->pool_N.n, c->poison);
}

// kernel parameters with the pool sizes current at this launch (LPB_CHECKS bounds)
DevParams dparams(const locpir_b200_ctx* c)
{
    DevParams d = c->dp;
    d.pool_slots = c->pool_slots;
    d.scratch_slots = c->pool_N.n / c->dp.N_stride;
    d.ext_a = c->ext_a;
    d.ext_b = c->ext_b;
    d.ext_rows = c->ext_rows;
    return d;
}

int fail(locpir_b200_ctx* c, int code, const std::string& msg)
{
    if (c)
        c->err = msg;
    return code;
}

template <class F>
int guarded(locpir_b200_ctx* c, F&& f)
{
    if (!c)
        return LOCPIR_B200_EINVAL;
    try {
        f();
        return LOCPIR_B200_OK;
    } catch (const std::invalid_argument& e) {
        return fail(c, LOCPIR_B200_EINVAL, e.what());
    } catch (const std::logic_error& e) {
        return fail(c, LOCPIR_B200_ELOGIC, e.what());
    } catch (const CudaError& e) {
        return fail(c, LOCPIR_B200_ECUDA, e.what());
    } catch (const std::bad_alloc&) {
        return fail(c, LOCPIR_B200_ENOMEM, "out of host memory");
    } catch (const std::exception& e) {
        return fail(c, LOCPIR_B200_ECUDA, e.what());
    }
}

// Transform tables: the same values as the oracle contract (oracle/tfhe_oracle.c
// or_fft2_make_tables, the same libm calls in long double, rounded to double):
//   forward tree node v (stage s, block b = v - 2^s): twiddle psi^(E[v]/2) as
//     (cos, tan), E[1] = N/2, children E/2 and E/2 + N (mod 2N), psi = e^{i pi / N};
//   inverse: W^e = e^{2 pi i e / M} (e < M/2, W[e + M/4] = i W[e] exactly) and the
//     base (cos, tan) of W^e, e < M/4;
//   twist psi^j in factored form cmul(psi^(j mod 64), psi^(j - j mod 64)).
// Per-thread tables [entry][t] for the 64-thread transform (fft.cuh FwdTw / InvTw).
struct Tables {
    std::vector<double2> fwd, inv, tw;  // [8][64], [8][64], [512]
    double2 fwd0[4], inv4, twq[8];
};

void ct_of(long num, long den, double& c, double& t)
{
    const long double pi = 3.141592653589793238462643383279502884L;
    if (num == 0) {
        c = 1.0;
        t = 0.0;
        return;
    }
    if (4 * num == den) {  // pi/4: tan = 1 exactly
        c = (double)cosl(pi / 4.0L);
        t = 1.0;
        return;
    }
    const long double th = pi * (long double)num / (long double)den;
    c = (double)cosl(th);
    t = (double)tanl(th);
}

Tables make_tables(uint32_t N)
{
    const uint32_t M = N / 2;  // 512
    Tables T;
    std::vector<uint32_t> E(2 * M);
    E[1] = N / 2;
    for (uint32_t v = 1; v < M; v++) {
        E[2 * v] = (E[v] / 2) % (2 * N);
        E[2 * v + 1] = (E[v] / 2 + N) % (2 * N);
    }
    std::vector<double2> node(M);
    for (uint32_t v = 1; v < M; v++)
        ct_of((long)(E[v] / 2), (long)N, node[v].x, node[v].y);
    const long double pi = 3.141592653589793238462643383279502884L;
    std::vector<double2> W(M / 2), ic(M / 4);
    for (uint32_t e = 0; e < M / 4; e++) {
        double re = 1.0, im = 0.0;
        if (e) {
            re = (double)cosl(2.0L * pi * (long double)e / (long double)M);
            im = (double)sinl(2.0L * pi * (long double)e / (long double)M);
        }
        W[e] = make_double2(re, im);
        W[e + M / 4] = make_double2(-im, re);
        ct_of(2 * (long)e, (long)M, ic[e].x, ic[e].y);
    }
    auto icj = [&](uint32_t e) { return make_double2(ic[e].x, -ic[e].y); };  // conj: -tan
    auto wcj = [&](uint32_t e) { return make_double2(W[e].x, -W[e].y); };
    T.fwd.assign(8 * 64, make_double2(0, 0));
    T.inv.assign(8 * 64, make_double2(0, 0));
    for (int t = 0; t < 64; t++) {
        const int k = t >> 3, r = t & 7;
        const double2 f[8] = {node[8 + k],   node[16 + 2 * k],  node[32 + 4 * k],
                              node[32 + 4 * k + 2], node[64 + t], node[128 + 2 * t],
                              node[256 + 4 * t], node[256 + 4 * t + 2]};
        const double2 g[8] = {wcj(32 * r), icj(16 * r), icj(8 * r), icj(8 * r + 64),
                              wcj(4 * t),  icj(2 * t),  icj(t),     icj(t + 64)};
        for (int e = 0; e < 8; e++) {
            T.fwd[e * 64 + t] = f[e];
            T.inv[e * 64 + t] = g[e];
        }
    }
    T.fwd0[0] = node[1];
    T.fwd0[1] = node[2];
    T.fwd0[2] = node[4];
    T.fwd0[3] = node[6];
    T.inv4 = icj(64);
    // twist psi^j (psi = e^{i pi / N}), factored as the kernels form it on the fly
    T.tw.assign(M, make_double2(0, 0));
    const double dpi = 3.14159265358979323846;
    for (uint32_t j = 0; j < M; j++)
        T.tw[j] = make_double2(j == 0 ? 1.0 : std::cos(dpi * (double)j / (double)N),
                               j == 0 ? 0.0 : std::sin(dpi * (double)j / (double)N));
    for (uint32_t j = M; j-- > 0;) {
        const uint32_t lo = j & 63u, hi = j & ~63u;
        if (lo && hi) {
            const double2 x = T.tw[lo], w = T.tw[hi];
            T.tw[j] = make_double2(std::fma(x.x, w.x, -(x.y * w.y)), std::fma(x.x, w.y, x.y * w.x));
        }
    }
    for (int q = 0; q < 8; q++)
        T.twq[q] = T.tw[64 * q];
    return T;
}

FftTabs tabs(const locpir_b200_ctx* c) { return FftTabs{c->ftw.p, c->itw.p, c->TW.p}; }

// contexts per device that hold a persisting-L2 BK window
int persist_users(int device, int delta)
{
    static std::mutex mu;
    static std::map<int, int> users;
    std::lock_guard<std::mutex> g(mu);
    return users[device] += delta;
}

void need_keys(locpir_b200_ctx* c)
{
    if (!c->have_keys)
        throw std::logic_error("bootstrapping and key-switching keys are not uploaded");
}

void check_owned(const locpir_b200_ctx* c, uint64_t slot_end)
{
    if (!c->server_calls && slot_end > c->server_base)
        throw std::invalid_argument("pool slots from " + std::to_string(c->server_base) +
                                    " on are owned by the batching server on this context");
}

void check_pool(locpir_b200_ctx* c, uint64_t first, uint64_t count)
{
    if (first + count > c->pool_slots || first + count < first)
        throw std::invalid_argument("pool slot range out of bounds");
    check_owned(c, first + count);
}

void timed_begin(locpir_b200_ctx* c, int k)
{
    if (!c->timing)
        return;
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, c->stream));
    c->timer.ev[k].push_back(e);
}
void timed_end(locpir_b200_ctx* c, int k)
{
    if (!c->timing)
        return;
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, c->stream));
    c->timer.ev[k].push_back(e);
    c->timer.launches[k]++;
}

void launch_br(locpir_b200_ctx* c, const BrItem* items, uint32_t count)
{
    if (!count)
        return;
    timed_begin(c, 0);
    const uint32_t mu = 0x20000000u;
    const FftTabs tb = tabs(c);
    if (c->small_levels && count <= (uint32_t)c->num_sms) {
        if (c->p.bk_l == 3 && c->p.bk_bgbit == 7)
            k_blind_rotate_lat<3, 7><<<count, 128 * 3, kLatSmemBytes<3>, c->stream>>>(
                dparams(c), items, c->pool_n.p, c->pool_N.p, c->bkf.p, tb, mu);
        else if (c->p.bk_l == 2 && c->p.bk_bgbit == 10)
            k_blind_rotate_lat<2, 10><<<count, 128 * 2, kLatSmemBytes<2>, c->stream>>>(
                dparams(c), items, c->pool_n.p, c->pool_N.p, c->bkf.p, tb, mu);
        else
            throw std::invalid_argument("no blind-rotate kernel instantiated for this (l, Bgbit)");
    } else {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(count);
        cfg.blockDim = dim3(64);
        cfg.stream = c->stream;
        cudaLaunchAttribute attr[1];
        if (c->have_window) {  // keep BK_freq L2-resident for this launch
            attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
            attr[0].val.accessPolicyWindow = c->bk_window;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
        }
        const uint32_t* pn = c->pool_n.p;
        uint32_t* pN = c->pool_N.p;
        const double2* bk = c->bkf.p;
        if (c->p.bk_l == 3 && c->p.bk_bgbit == 7)
            CK(cudaLaunchKernelEx(&cfg, k_blind_rotate<3, 7>, dparams(c), items, pn, pN, bk, tb, mu,
                                  (unsigned long long*)nullptr));
        else if (c->p.bk_l == 2 && c->p.bk_bgbit == 10)
            CK(cudaLaunchKernelEx(&cfg, k_blind_rotate<2, 10>, dparams(c), items, pn, pN, bk, tb, mu,
                                  (unsigned long long*)nullptr));
        else
            throw std::invalid_argument("no blind-rotate kernel instantiated for this (l, Bgbit)");
    }
    CK(cudaGetLastError());
    timed_end(c, 0);
}

void launch_ks(locpir_b200_ctx* c, const KsItem* items, uint32_t count)
{
    if (!count)
        return;
    timed_begin(c, 1);
    if (c->ks_tc && c->kskt_tiles && count >= KT_MIN_COUNT) {
        // K2t: N tiles fast in the grid, one M tile (256 ciphertexts) per grid row
        k_keyswitch_tc<<<dim3(c->kskt_tiles, (count + KT_M * KT_HALVES - 1) / (KT_M * KT_HALVES)),
                         KT_THREADS, KT_SMEM, c->stream>>>(dparams(c), items, count, c->pool_N.p,
                                                           c->pool_n.p, c->kskt.p);
        CK(cudaGetLastError());
        timed_end(c, 1);
        return;
    }
    const uint32_t blocks = (count + KS_CT - 1) / KS_CT;
    if (c->small_levels && blocks < (uint32_t)c->num_sms / 2) {
        c->ks_partial.reserve((size_t)count * KS_SPLIT * c->dp.n_stride, c->stream, false);
        k_keyswitch_split<<<dim3(count, KS_SPLIT), KS_THREADS, 0, c->stream>>>(
            dparams(c), items, c->pool_N.p, c->ksk.p, c->ks_partial.p);
        k_ks_reduce<<<count, KS_THREADS, 0, c->stream>>>(dparams(c), items, c->pool_N.p,
                                                          c->ks_partial.p, c->pool_n.p);
        CK(cudaGetLastError());
        timed_end(c, 1);
        return;
    }
    const size_t smem = (size_t)KS_CT * c->p.N * sizeof(uint16_t);
    k_keyswitch<<<blocks, KS_THREADS, smem, c->stream>>>(dparams(c), items, count, c->pool_N.p,
                                                         c->pool_n.p, c->ksk.p);
    CK(cudaGetLastError());
    timed_end(c, 1);
}

void launch_lin(locpir_b200_ctx* c, const LinItem* items, uint32_t count)
{
    if (!count)
        return;
    timed_begin(c, 2);
    const uint64_t total = (uint64_t)count * (c->p.n + 1);
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((total + 255) / 256, 148ull * 16);
    k_linear<<<blocks, 256, 0, c->stream>>>(dparams(c), items, count, c->pool_n.p);
    CK(cudaGetLastError());
    timed_end(c, 2);
}

void validate_slots(locpir_b200_ctx* c, const locpir_b200_gate_op* ops, uint64_t count)
{
    for (uint64_t g = 0; g < count; g++) {
        const auto& op = ops[g];
        for (uint32_t s : {op.in0, op.in1, op.in2})
            if (s != SLOT_NONE && s >= c->pool_slots &&
                !(op.kind == LOCPIR_B200_CONST && s == op.in0))
                throw std::invalid_argument("operand slot " + std::to_string(s) +
                                            " outside the pool");
        if (op.out >= c->pool_slots)
            throw std::invalid_argument("output slot outside the pool");
        for (uint32_t s : {op.in0, op.in1, op.in2, op.out})
            if (s != SLOT_NONE && !(op.kind == LOCPIR_B200_CONST && s == op.in0 && s != op.out))
                check_owned(c, (uint64_t)s + 1);
    }
}

}  // namespace

// A planned program: per-wave item ranges in device memory.
struct locpir_b200_program {
    Plan plan;
    int device = 0;
    DevBuf<BrItem> br;
    DevBuf<KsItem> ks;
    DevBuf<LinItem> lin;
    std::vector<size_t> ob, ok, ol;  // per-wave offsets
    uint64_t kernels = 0;
    // CUDA graph of the launch sequence, valid for the device buffers in `sig`
    cudaGraphExec_t exec = nullptr;
    std::vector<const void*> sig;
    uint64_t launches = 0;
    ~locpir_b200_program()
    {
        if (exec)
            cudaGraphExecDestroy(exec);
    }
};

namespace {

void program_upload(locpir_b200_ctx* c, locpir_b200_program* pr, BrItem* hb, KsItem* hk,
                    LinItem* hl, DevBuf<BrItem>& db, DevBuf<KsItem>& dk, DevBuf<LinItem>& dl)
{
    const Plan& P = pr->plan;
    size_t ob = 0, ok = 0, ol = 0;
    pr->ob.clear();
    pr->ok.clear();
    pr->ol.clear();
    pr->kernels = 0;
    for (uint32_t w = 0; w < P.waves(); w++) {
        pr->ob.push_back(ob);
        pr->ok.push_back(ok);
        pr->ol.push_back(ol);
        std::copy(P.br[w].begin(), P.br[w].end(), hb + ob);
        std::copy(P.ks[w].begin(), P.ks[w].end(), hk + ok);
        std::copy(P.lin[w].begin(), P.lin[w].end(), hl + ol);
        ob += P.br[w].size();
        ok += P.ks[w].size();
        ol += P.lin[w].size();
        pr->kernels += !P.br[w].empty() + !P.ks[w].empty() + !P.lin[w].empty();
    }
    db.reserve(ob + 1, c->stream, false);
    dk.reserve(ok + 1, c->stream, false);
    dl.reserve(ol + 1, c->stream, false);
    if (ob)
        CK(cudaMemcpyAsync(db.p, hb, ob * sizeof(BrItem), cudaMemcpyHostToDevice, c->stream));
    if (ok)
        CK(cudaMemcpyAsync(dk.p, hk, ok * sizeof(KsItem), cudaMemcpyHostToDevice, c->stream));
    if (ol)
        CK(cudaMemcpyAsync(dl.p, hl, ol * sizeof(LinItem), cudaMemcpyHostToDevice, c->stream));
}

void program_kernels(locpir_b200_ctx* c, const locpir_b200_program* pr, const BrItem* db,
                     const KsItem* dk, const LinItem* dl)
{
    const Plan& P = pr->plan;
    for (uint32_t w = 0; w < P.waves(); w++) {
        launch_lin(c, dl + pr->ol[w], (uint32_t)P.lin[w].size());
        launch_br(c, db + pr->ob[w], (uint32_t)P.br[w].size());
        launch_ks(c, dk + pr->ok[w], (uint32_t)P.ks[w].size());
    }
}

void program_prepare(locpir_b200_ctx* c, const locpir_b200_program* pr)
{
    const Plan& P = pr->plan;
    if (P.n_br)
        need_keys(c);
    if (P.scratch > c->scratch_slots) {
        grow_scratch(c, P.scratch);
        c->scratch_slots = c->pool_N.n / c->dp.N_stride;
    }
}

void program_enqueue(locpir_b200_ctx* c, const locpir_b200_program* pr, const BrItem* db,
                     const KsItem* dk, const LinItem* dl)
{
    program_prepare(c, pr);
    program_kernels(c, pr, db, dk, dl);
    for (int i = 0; i < 9; i++)
        c->counters[i] += pr->plan.counts[i];
}

// Every device pointer a captured launch sequence bakes in.
std::vector<const void*> graph_signature(const locpir_b200_ctx* c)
{
    return {c->pool_n.p, c->pool_N.p, c->ks_partial.p, c->bkf.p, c->ksk.p, c->kskt.p,
            c->ftw.p,    c->itw.p,    c->TW.p,         (const void*)c->stream};
}

size_t plan_items(const Plan& P, size_t& nb, size_t& nk, size_t& nl)
{
    nb = nk = nl = 0;
    for (uint32_t w = 0; w < P.waves(); w++) {
        nb += P.br[w].size();
        nk += P.ks[w].size();
        nl += P.lin[w].size();
    }
    return nb + nk + nl;
}

void execute(locpir_b200_ctx* c, const locpir_b200_gate_op* ops, uint64_t count)
{
    validate_slots(c, ops, count);
    locpir_b200_program pr;
    pr.plan = build_plan(ops, count);  // throws invalid_argument on malformed programs
    size_t nb, nk, nl;
    plan_items(pr.plan, nb, nk, nl);
    CK(cudaStreamSynchronize(c->stream));  // pinned staging may still feed an earlier copy
    c->h_br.reserve(nb + 1);
    c->h_ks.reserve(nk + 1);
    c->h_lin.reserve(nl + 1);
    program_upload(c, &pr, c->h_br.p, c->h_ks.p, c->h_lin.p, c->d_br, c->d_ks, c->d_lin);
    program_enqueue(c, &pr, c->d_br.p, c->d_ks.p, c->d_lin.p);
}

void pool_copy(locpir_b200_ctx* c, uint64_t first, uint64_t count, const uint32_t* src,
               uint32_t* dst, cudaMemcpyKind kind, bool to_pool)
{
    check_pool(c, first, count);
    if (!count)
        return;
    const size_t wb = (size_t)(c->p.n + 1) * 4, pb = (size_t)c->dp.n_stride * 4;
    if (to_pool && kind == cudaMemcpyHostToDevice && count >= 256) {
        // one 1-D copy into a packed staging buffer + an HBM-speed repack kernel
        c->h2d_stage.reserve((size_t)count * (c->p.n + 1), c->stream, false);
        CK(cudaMemcpyAsync(c->h2d_stage.p, src, (size_t)count * wb, kind, c->stream));
        k_repack_rows<<<c->num_sms * 8, 256, 0, c->stream>>>(dparams(c), c->h2d_stage.p, count,
                                                             c->pool_n.p + first * c->dp.n_stride);
        CK(cudaGetLastError());
    } else if (to_pool) {
        CK(cudaMemcpy2DAsync(c->pool_n.p + first * c->dp.n_stride, pb, src, wb, wb, count, kind,
                             c->stream));
    } else if (kind == cudaMemcpyDeviceToHost && count >= 256) {
        c->d2h_stage.reserve((size_t)count * (c->p.n + 1), c->stream, false);
        k_pack_rows<<<c->num_sms * 8, 256, 0, c->stream>>>(dparams(c), c->pool_n.p + first * c->dp.n_stride,
                                                           count, c->d2h_stage.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(dst, c->d2h_stage.p, (size_t)count * wb, kind, c->stream));
    } else {
        CK(cudaMemcpy2DAsync(dst, wb, c->pool_n.p + first * c->dp.n_stride, pb, wb, count, kind,
                             c->stream));
    }
}

// Device address of a pinned, device-mapped host buffer (cudaHostAlloc / pinned torch
// tensors under unified addressing), or nullptr for pageable memory.
const uint32_t* mapped_host(const uint32_t* p)
{
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? static_cast<const uint32_t*>(at.devicePointer) : nullptr;
}

// gate_batch_host on pinned inputs: the blind rotation's prologue reads each gate's two
// input rows straight from the caller's buffers over PCIe (slots SLOT_EXT_A / _B), so no
// host-to-device copy and no repack precede the first K1 wave; one level, so the items are
// built directly (no planner).  Outputs land in pool slots [0, count) and are packed and
// copied back as in the copy path.
void gate_batch_zero_copy(locpir_b200_ctx* c, uint32_t kind, const GateForm& f,
                          const uint32_t* da, const uint32_t* db, uint32_t* out, uint64_t count)
{
    need_keys(c);
    check_owned(c, count);
    if (c->pool_slots < count) {
        int rc = locpir_b200_pool_reserve(c, count);
        if (rc)
            throw CudaError(c->err);
    }
    if (count > c->scratch_slots) {
        grow_scratch(c, count);
        c->scratch_slots = c->pool_N.n / c->dp.N_stride;
    }
    CK(cudaStreamSynchronize(c->stream));  // pinned staging may still feed an earlier copy
    c->h_br.reserve(count + 1);
    c->h_ks.reserve(count + 1);
    for (uint64_t g = 0; g < count; g++) {
        c->h_br.p[g] = {SLOT_EXT_A | (uint32_t)g, SLOT_EXT_B | (uint32_t)g, f.c0, f.c1, f.off,
                        (uint32_t)g, SLOT_NONE, 0};
        c->h_ks.p[g] = {(uint32_t)g, SLOT_NONE, 0u, (uint32_t)g};
    }
    c->d_br.reserve(count + 1, c->stream, false);
    c->d_ks.reserve(count + 1, c->stream, false);
    CK(cudaMemcpyAsync(c->d_br.p, c->h_br.p, count * sizeof(BrItem), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaMemcpyAsync(c->d_ks.p, c->h_ks.p, count * sizeof(KsItem), cudaMemcpyHostToDevice,
                       c->stream));
    c->ext_a = da;
    c->ext_b = db;
    c->ext_rows = (uint32_t)count;
    try {
        launch_br(c, c->d_br.p, (uint32_t)count);
    } catch (...) {
        c->ext_a = c->ext_b = nullptr;
        c->ext_rows = 0;
        throw;
    }
    c->ext_a = c->ext_b = nullptr;
    c->ext_rows = 0;
    launch_ks(c, c->d_ks.p, (uint32_t)count);
    static const int cidx[] = {0, 1, 2, 3, 6, -1, -1, 7, -1, -1, 0, 1};  // as Plan::counts
    c->counters[cidx[kind]] += count;
    c->counters[8] += count;
    pool_copy(c, 0, count, nullptr, out, cudaMemcpyDeviceToHost, false);
}

// QUERY framing check in the order the reference's ByteReader consumes the bytes
// (handle_query, protocol.hpp:401-407: read_word x2 + expect_done; codec.hpp:180-193;
// bytes.hpp:66-130), throwing the reference's DecodeError messages as invalid_argument.
void check_query(uint32_t n, const uint8_t* b, uint64_t len, uint32_t l)
{
    const uint64_t S = 4ull * (n + 1);
    uint64_t pos = 0;
    for (int w = 0; w < 2; w++) {
        if (len - pos < 1)
            throw std::invalid_argument("truncated input: need 1 bytes, have " +
                                        std::to_string(len - pos));
        const uint32_t lw = b[pos++];
        if (lw != l)
            throw std::invalid_argument("cipher word length " + std::to_string(lw) +
                                        " does not match negotiated format l=" +
                                        std::to_string(l));
        if (len - pos < (uint64_t)l * S)
            throw std::invalid_argument("truncated input: need 4 bytes, have " +
                                        std::to_string((len - pos) % 4));
        pos += (uint64_t)l * S;
    }
    if (pos != len)
        throw std::invalid_argument("trailing bytes: " + std::to_string(len - pos));
}

}  // namespace

extern "C" {

int locpir_b200_ctx_create(const locpir_b200_params* p, int device, void* stream,
                           locpir_b200_ctx** out)
{
    if (!p || !out || !locpir_b200_bk_words(p))
        return LOCPIR_B200_EINVAL;
    // the device kernels are built for n <= 636 (K2 column coverage, abar arrays) and the
    // two gadget shapes of the BASELINE parameter sets
    if (p->n > MAX_CTX_N || !((p->bk_l == 3 && p->bk_bgbit == 7) || (p->bk_l == 2 && p->bk_bgbit == 10)))
        return LOCPIR_B200_EINVAL;
    static_assert(KS_THREADS * KS_COLS >= ((MAX_CTX_N + 1 + 3) & ~3u), "K2 column coverage");
    *out = nullptr;
    auto c = std::make_unique<locpir_b200_ctx>();
    c->p = *p;
    c->device = device;
    const uint32_t ns = (p->n + 1 + 3) & ~3u;
    c->dp = {p->n, p->N, p->bk_l, p->bk_bgbit, p->ks_t, p->ks_basebit, ns, p->N + 4, 0, 0};
    int rc = guarded(c.get(), [&] {
        CK(cudaSetDevice(device));
        CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        if (stream) {
            c->stream = (cudaStream_t)stream;
        } else {
            CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->own_stream = true;
        }
        const Tables T = make_tables(p->N);
        c->ftw.reserve(T.fwd.size(), c->stream, false);
        c->itw.reserve(T.inv.size(), c->stream, false);
        c->TW.reserve(T.tw.size(), c->stream, false);
        CK(cudaMemcpy(c->ftw.p, T.fwd.data(), T.fwd.size() * sizeof(double2), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->itw.p, T.inv.data(), T.inv.size() * sizeof(double2), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(c->TW.p, T.tw.data(), T.tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
        CK(cudaMemcpyToSymbol(c_twq, T.twq, sizeof(T.twq)));
        CK(cudaMemcpyToSymbol(c_fwd0, T.fwd0, sizeof(T.fwd0)));
        CK(cudaMemcpyToSymbol(c_inv4, &T.inv4, sizeof(T.inv4)));
        CK(cudaFuncSetAttribute(k_keyswitch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(KS_CT * p->N * sizeof(uint16_t))));
        CK(cudaFuncSetAttribute(k_keyswitch_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)KT_SMEM));
        if (const char* kt = getenv("LOCPIR_B200_KSTC"))
            c->ks_tc = strcmp(kt, "0") != 0;
        CK(cudaFuncSetAttribute(k_blind_rotate_lat<3, 7>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLatSmemBytes<3>));
        CK(cudaFuncSetAttribute(k_blind_rotate_lat<2, 10>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLatSmemBytes<2>));
        if (const char* lp = getenv("LOCPIR_B200_L2PERSIST"))
            c->l2_persist = strcmp(lp, "0") != 0;
        if (const char* sl = getenv("LOCPIR_B200_SMALL"))
            c->small_levels = strcmp(sl, "0") != 0;
        if (const char* gr = getenv("LOCPIR_B200_GRAPH"))
            c->use_graphs = strcmp(gr, "0") != 0;
        if (const char* zc = getenv("LOCPIR_B200_ZEROCOPY"))
            c->zero_copy = strcmp(zc, "0") != 0;
        if (const char* po = getenv("LOCPIR_B200_POISON"); po && *po) {
            c->poison = (uint32_t)strtoul(po, nullptr, 0);
            c->poison_set = true;
            CK(cudaMemcpyToSymbol(c_poison, &c->poison, sizeof(uint32_t)));
        }
    });
    if (rc != LOCPIR_B200_OK) {
        fprintf(stderr, "locpir_b200_ctx_create: %s\n", c->err.c_str());
        if (c->own_stream && c->stream)
            cudaStreamDestroy(c->stream);
        return rc;
    }
    *out = c.release();
    return LOCPIR_B200_OK;
}

void locpir_b200_ctx_destroy(locpir_b200_ctx* c)
{
    if (!c)
        return;
    cudaSetDevice(c->device);
    if (c->stream)
        cudaStreamSynchronize(c->stream);
    if (c->have_window && persist_users(c->device, -1) == 0) {
        // the last context with a BK window: hand the persisting L2 back
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
        cudaGetLastError();
    }
    for (auto& v : c->timer.ev)
        for (auto e : v)
            cudaEventDestroy(e);
    if (c->own_stream && c->stream)
        cudaStreamDestroy(c->stream);
    delete c;
}

const char* locpir_b200_last_error(const locpir_b200_ctx* c) { return c ? c->err.c_str() : ""; }

void* locpir_b200_stream(const locpir_b200_ctx* c) { return c ? (void*)c->stream : nullptr; }

int locpir_b200_upload_keys(locpir_b200_ctx* c, const uint32_t* bk, const uint32_t* ksk,
                            int on_device)
{
    return guarded(c, [&] {
        if (!bk || !ksk)
            throw std::invalid_argument("null key pointer");
        CK(cudaSetDevice(c->device));
        const size_t bkw = locpir_b200_bk_words(&c->p);
        const uint32_t rows = 2 * c->p.bk_l;
        const size_t polys = (size_t)c->p.n * rows * 2;
        DevBuf<uint32_t> tmp;
        const uint32_t* dbk = bk;
        if (!on_device) {
            tmp.reserve(bkw, c->stream, false);
            CK(cudaMemcpyAsync(tmp.p, bk, bkw * 4, cudaMemcpyHostToDevice, c->stream));
            dbk = tmp.p;
        }
        c->bkf.reserve(polys * FFT_M, c->stream, false);
        k_bk_to_freq<<<(uint32_t)polys, 64, 0, c->stream>>>(dbk, c->bkf.p, tabs(c));
        CK(cudaGetLastError());
        // KSK rows padded to n_stride words (zero padding)
        const size_t rows_ks = (size_t)c->p.N * c->p.ks_t * ((1u << c->p.ks_basebit) - 1);
        c->ksk.reserve(rows_ks * c->dp.n_stride, c->stream, false);
        CK(cudaMemsetAsync(c->ksk.p, 0, rows_ks * c->dp.n_stride * 4, c->stream));
        CK(cudaMemcpy2DAsync(c->ksk.p, (size_t)c->dp.n_stride * 4, ksk, (size_t)(c->p.n + 1) * 4,
                             (size_t)(c->p.n + 1) * 4, rows_ks,
                             on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                             c->stream));
        // K2t: the KSK as byte-sliced tiles for the INT8 tensor-core key switch
        if (c->p.ks_t == 8 && c->p.ks_basebit == 2 && c->p.N * 8 * 3 % (2 * KT_KC) == 0) {  // stage pairs
            c->kskt_tiles = (c->dp.n_stride * 4 + KT_N - 1) / KT_N;
            const size_t chunks =
                (size_t)c->kskt_tiles * (c->p.N * c->p.ks_t * 3 / KT_KC) * KT_CHUNKS * KT_N;
            c->kskt.reserve(chunks, c->stream, false);
            k_ksk_to_tc<<<c->num_sms * 16, 256, 0, c->stream>>>(dparams(c), c->ksk.p, c->kskt_tiles,
                                                                c->kskt.p);
            CK(cudaGetLastError());
        }
        CK(cudaStreamSynchronize(c->stream));
        c->have_keys = true;
        // Keep the frequency-domain BK resident in L2 (persisting access window, attached
        // to every K1 launch): at cfg2 scale the blind-rotate CTAs sweep all 62 MB of it out
        // of step with each other.
        if (c->l2_persist) {
            int maxp = 0, maxw = 0;
            cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, c->device);
            cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
            const size_t bytes = c->bkf.n * sizeof(double2);
            if (maxp > 0 && maxw > 0) {
                if (!c->have_window && persist_users(c->device, +1) == 1)
                    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp);
                cudaAccessPolicyWindow& w = c->bk_window;
                w.base_ptr = c->bkf.p;
                w.num_bytes = std::min<size_t>(bytes, maxw);
                w.hitRatio = std::min(1.0f, (float)std::min<size_t>(bytes, maxp) / (float)w.num_bytes);
                w.hitProp = cudaAccessPropertyPersisting;
                w.missProp = cudaAccessPropertyStreaming;
                c->have_window = true;
                cudaGetLastError();
            }
        }
    });
}

int locpir_b200_pool_reserve(locpir_b200_ctx* c, uint64_t slots)
{
    return guarded(c, [&] {
        CK(cudaSetDevice(c->device));
        if (slots <= c->pool_slots)
            return;
        c->pool_n.reserve((size_t)slots * c->dp.n_stride, c->stream, true);
        const uint64_t old = c->pool_slots;
        c->pool_slots = c->pool_n.n / c->dp.n_stride;
        fill_words(c, c->pool_n.p + old * c->dp.n_stride, (c->pool_slots - old) * c->dp.n_stride,
                   c->poison);
    });
}

uint64_t locpir_b200_pool_capacity(const locpir_b200_ctx* c) { return c ? c->pool_slots : 0; }

int locpir_b200_pool_h2d(locpir_b200_ctx* c, uint64_t first, uint64_t count, const uint32_t* host)
{
    return guarded(c, [&] {
        pool_copy(c, first, count, host, nullptr, cudaMemcpyHostToDevice, true);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int locpir_b200_pool_d2h(locpir_b200_ctx* c, uint64_t first, uint64_t count, uint32_t* host)
{
    return guarded(c, [&] {
        pool_copy(c, first, count, nullptr, host, cudaMemcpyDeviceToHost, false);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int locpir_b200_pool_load_device(locpir_b200_ctx* c, uint64_t first, uint64_t count,
                                 const uint32_t* dev)
{
    return guarded(c, [&] { pool_copy(c, first, count, dev, nullptr, cudaMemcpyDeviceToDevice, true); });
}

int locpir_b200_pool_store_device(locpir_b200_ctx* c, uint64_t first, uint64_t count,
                                  uint32_t* dev)
{
    return guarded(c, [&] { pool_copy(c, first, count, nullptr, dev, cudaMemcpyDeviceToDevice, false); });
}

int locpir_b200_run(locpir_b200_ctx* c, const locpir_b200_gate_op* ops, uint64_t count)
{
    return guarded(c, [&] {
        if (count && !ops)
            throw std::invalid_argument("null program");
        CK(cudaSetDevice(c->device));
        execute(c, ops, count);
    });
}

int locpir_b200_eval_level(locpir_b200_ctx* c, const locpir_b200_gate_op* ops, uint64_t count)
{
    return guarded(c, [&] {
        if (count && !ops)
            throw std::invalid_argument("null program");
        Plan P = build_plan(ops, count);
        if (P.waves() > 1)
            throw std::invalid_argument("eval_level: gates of one level must be independent");
        CK(cudaSetDevice(c->device));
        execute(c, ops, count);
    });
}

int locpir_b200_sync(locpir_b200_ctx* c)
{
    return guarded(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int locpir_b200_program_create(locpir_b200_ctx* c, const locpir_b200_gate_op* ops,
                               uint64_t count, locpir_b200_program** out)
{
    return guarded(c, [&] {
        if (!out || (count && !ops))
            throw std::invalid_argument("bad program arguments");
        CK(cudaSetDevice(c->device));
        validate_slots(c, ops, count);
        auto pr = std::make_unique<locpir_b200_program>();
        pr->plan = build_plan(ops, count);
        pr->device = c->device;
        size_t nb, nk, nl;
        plan_items(pr->plan, nb, nk, nl);
        std::vector<BrItem> hb(nb + 1);
        std::vector<KsItem> hk(nk + 1);
        std::vector<LinItem> hl(nl + 1);
        program_upload(c, pr.get(), hb.data(), hk.data(), hl.data(), pr->br, pr->ks, pr->lin);
        CK(cudaStreamSynchronize(c->stream));
        // drop the host-side lists; keep sizes for launching
        *out = pr.release();
    });
}

int locpir_b200_program_launch(locpir_b200_ctx* c, locpir_b200_program* pr)
{
    return guarded(c, [&] {
        if (!pr)
            throw std::invalid_argument("null program");
        // The first launch runs directly (it also sizes every buffer: no allocation may
        // happen under capture); later launches replay a CUDA graph of the whole level
        // sequence, re-captured whenever a device buffer moved.  Timing mode (per-kernel
        // events) and LOCPIR_B200_GRAPH=0 launch directly.
        if (!c->use_graphs || c->timing || pr->launches == 0 || pr->plan.waves() == 0) {
            program_enqueue(c, pr, pr->br.p, pr->ks.p, pr->lin.p);
            pr->launches++;
            return;
        }
        program_prepare(c, pr);
        const auto sig = graph_signature(c);
        if (!pr->exec || pr->sig != sig) {
            if (pr->exec) {
                CK(cudaGraphExecDestroy(pr->exec));
                pr->exec = nullptr;
            }
            cudaGraph_t graph = nullptr;
            CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            try {
                program_kernels(c, pr, pr->br.p, pr->ks.p, pr->lin.p);
            } catch (...) {
                cudaStreamEndCapture(c->stream, &graph);
                if (graph)
                    cudaGraphDestroy(graph);
                throw;
            }
            CK(cudaStreamEndCapture(c->stream, &graph));
            const cudaError_t e = cudaGraphInstantiate(&pr->exec, graph, 0);
            cudaGraphDestroy(graph);
            CK(e);
            pr->sig = sig;
        }
        CK(cudaGraphLaunch(pr->exec, c->stream));
        for (int i = 0; i < 9; i++)
            c->counters[i] += pr->plan.counts[i];
        pr->launches++;
    });
}

int locpir_b200_program_prepare(locpir_b200_ctx* c, locpir_b200_program* pr)
{
    return guarded(c, [&] {
        if (!pr)
            throw std::invalid_argument("null program");
        program_prepare(c, pr);  // keys present, N-dim scratch sized: no allocation at launch
    });
}

uint64_t locpir_b200_program_kernels(const locpir_b200_program* pr) { return pr ? pr->kernels : 0; }

void locpir_b200_program_destroy(locpir_b200_program* pr)
{
    if (!pr)
        return;
    cudaSetDevice(pr->device);
    cudaDeviceSynchronize();
    delete pr;
}

int locpir_b200_plan(const locpir_b200_gate_op* ops, uint64_t count, uint32_t* levels,
                     uint64_t* blind_rotations, uint64_t* key_switches)
{
    try {
        Plan P = build_plan(ops, count);
        if (levels) {  // bootstrap levels (a trailing wave of free linear ops is not one)
            uint32_t lv = 0;
            for (uint32_t w = 0; w < P.waves(); w++)
                lv += !P.br[w].empty();
            *levels = lv;
        }
        if (blind_rotations)
            *blind_rotations = P.n_br;
        if (key_switches)
            *key_switches = P.n_ks;
        return LOCPIR_B200_OK;
    } catch (const std::invalid_argument&) {
        return LOCPIR_B200_EINVAL;
    } catch (...) {
        return LOCPIR_B200_ELOGIC;
    }
}

int locpir_b200_counters(const locpir_b200_ctx* c, uint64_t out[9])
{
    if (!c || !out)
        return LOCPIR_B200_EINVAL;
    for (int i = 0; i < 9; i++)
        out[i] = c->counters[i];
    return LOCPIR_B200_OK;
}

int locpir_b200_counters_reset(locpir_b200_ctx* c)
{
    if (!c)
        return LOCPIR_B200_EINVAL;
    for (auto& x : c->counters)
        x = 0;
    return LOCPIR_B200_OK;
}

int locpir_b200_gate_batch_host(locpir_b200_ctx* c, uint32_t kind, const uint32_t* a,
                                const uint32_t* b, uint32_t* out, uint64_t count)
{
    return guarded(c, [&] {
        GateForm f;
        if (!gate_form(kind, f))
            throw std::invalid_argument("gate_batch_host takes a two-input bootstrapped gate");
        if (count >= (1ull << 30) || (count && (!a || !b || !out)))
            throw std::invalid_argument("bad batch");
        CK(cudaSetDevice(c->device));
        if (c->zero_copy && count >= 256 && count < (1ull << 29)) {
            const uint32_t* da = mapped_host(a);
            const uint32_t* db = mapped_host(b);
            if (da && db) {
                gate_batch_zero_copy(c, kind, f, da, db, out, count);
                CK(cudaStreamSynchronize(c->stream));
                return;
            }
        }
        if (c->pool_slots < 3 * count) {
            int rc = locpir_b200_pool_reserve(c, 3 * count);
            if (rc)
                throw CudaError(c->err);
        }
        pool_copy(c, 0, count, a, nullptr, cudaMemcpyHostToDevice, true);
        pool_copy(c, count, count, b, nullptr, cudaMemcpyHostToDevice, true);
        std::vector<locpir_b200_gate_op> ops(count);
        for (uint64_t g = 0; g < count; g++)
            ops[g] = {kind, (uint32_t)g, (uint32_t)(count + g), SLOT_NONE, (uint32_t)(2 * count + g)};
        execute(c, ops.data(), count);
        pool_copy(c, 2 * count, count, nullptr, out, cudaMemcpyDeviceToHost, false);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int locpir_b200_debug_blind_rotate(locpir_b200_ctx* c, const uint32_t* lwe_n, uint64_t count,
                                   uint32_t* out_N)
{
    return guarded(c, [&] {
        if (count && (!lwe_n || !out_N))
            throw std::invalid_argument("null buffer");
        need_keys(c);
        CK(cudaSetDevice(c->device));
        if (c->pool_slots < count) {
            int rc = locpir_b200_pool_reserve(c, count);
            if (rc)
                throw CudaError(c->err);
        }
        pool_copy(c, 0, count, lwe_n, nullptr, cudaMemcpyHostToDevice, true);
        std::vector<BrItem> items(count);
        for (uint64_t g = 0; g < count; g++)
            items[g] = {(uint32_t)g, SLOT_NONE, 1, 0, 0u, (uint32_t)g, SLOT_NONE, 0};
        if (count > c->scratch_slots) {
            grow_scratch(c, count);
            c->scratch_slots = c->pool_N.n / c->dp.N_stride;
        }
        DevBuf<BrItem> d;
        d.reserve(count + 1, c->stream, false);
        CK(cudaMemcpyAsync(d.p, items.data(), count * sizeof(BrItem), cudaMemcpyHostToDevice,
                           c->stream));
        launch_br(c, d.p, (uint32_t)count);
        CK(cudaMemcpy2DAsync(out_N, (size_t)(c->p.N + 1) * 4, c->pool_N.p, (size_t)c->dp.N_stride * 4,
                             (size_t)(c->p.N + 1) * 4, count, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int locpir_b200_debug_keyswitch(locpir_b200_ctx* c, const uint32_t* lwe_N, uint64_t count,
                                uint32_t* out_n)
{
    return guarded(c, [&] {
        if (count && (!lwe_N || !out_n))
            throw std::invalid_argument("null buffer");
        need_keys(c);
        CK(cudaSetDevice(c->device));
        if (c->pool_slots < count) {
            int rc = locpir_b200_pool_reserve(c, count);
            if (rc)
                throw CudaError(c->err);
        }
        if (count > c->scratch_slots) {
            grow_scratch(c, count);
            c->scratch_slots = c->pool_N.n / c->dp.N_stride;
        }
        CK(cudaMemcpy2DAsync(c->pool_N.p, (size_t)c->dp.N_stride * 4, lwe_N, (size_t)(c->p.N + 1) * 4,
                             (size_t)(c->p.N + 1) * 4, count, cudaMemcpyHostToDevice, c->stream));
        std::vector<KsItem> items(count);
        for (uint64_t g = 0; g < count; g++)
            items[g] = {(uint32_t)g, SLOT_NONE, 0u, (uint32_t)g};
        DevBuf<KsItem> d;
        d.reserve(count + 1, c->stream, false);
        CK(cudaMemcpyAsync(d.p, items.data(), count * sizeof(KsItem), cudaMemcpyHostToDevice,
                           c->stream));
        launch_ks(c, d.p, (uint32_t)count);
        pool_copy(c, 0, count, nullptr, out_n, cudaMemcpyDeviceToHost, false);
        CK(cudaStreamSynchronize(c->stream));
    });
}

uint64_t locpir_b200_loc_pir_scratch(uint32_t Q, uint32_t R, uint32_t l, uint32_t m)
{
    return loc_pir_scratch(Q, R, l, m);
}

static int loc_pir_program_impl(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                const uint32_t* x_slots, const uint32_t* y_slots,
                                const uint32_t* bnd_slots, const uint32_t* svc_slots,
                                const uint32_t* out_slots, uint64_t scratch_first, int xor_tree,
                                locpir_b200_gate_op* ops, uint64_t* count, int cmp)
{
    if (!count || !Q || !R || l < 2 || !m || !x_slots || !y_slots || !bnd_slots || !svc_slots ||
        !out_slots || xor_tree < 0 || xor_tree > 2)
        return LOCPIR_B200_EINVAL;
    try {
        std::vector<locpir_b200_gate_op> v;
        emit_loc_pir(v, Q, R, l, m, x_slots, y_slots, bnd_slots, svc_slots, out_slots,
                     scratch_first, xor_tree, cmp);
        if (ops) {
            if (*count < v.size())
                return LOCPIR_B200_EINVAL;
            std::copy(v.begin(), v.end(), ops);
        }
        *count = v.size();
        return LOCPIR_B200_OK;
    } catch (...) {
        return LOCPIR_B200_EINVAL;
    }
}

int locpir_b200_loc_pir_program(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                const uint32_t* x_slots, const uint32_t* y_slots,
                                const uint32_t* bnd_slots, const uint32_t* svc_slots,
                                const uint32_t* out_slots, uint64_t scratch_first, int xor_tree,
                                locpir_b200_gate_op* ops, uint64_t* count)
{
    return loc_pir_program_impl(Q, R, l, m, x_slots, y_slots, bnd_slots, svc_slots, out_slots,
                                scratch_first, xor_tree, ops, count, 0);
}

int locpir_b200_loc_pir_maj_program(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                    const uint32_t* x_slots, const uint32_t* y_slots,
                                    const uint32_t* bnd_slots, const uint32_t* svc_slots,
                                    const uint32_t* out_slots, uint64_t scratch_first,
                                    int xor_tree, locpir_b200_gate_op* ops, uint64_t* count)
{
    return loc_pir_program_impl(Q, R, l, m, x_slots, y_slots, bnd_slots, svc_slots, out_slots,
                                scratch_first, xor_tree, ops, count, 1);
}

int locpir_b200_loc_pir_program_ex(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                   const uint32_t* x_slots, const uint32_t* y_slots,
                                   const uint32_t* bnd_slots, const int64_t* boxes,
                                   const uint32_t* svc_slots, const uint32_t* out_slots,
                                   uint64_t scratch_first, int xor_tree, int comparator,
                                   locpir_b200_gate_op* ops, uint64_t* count)
{
    if (comparator < 0 || comparator > 2 || (!bnd_slots == !boxes))
        return LOCPIR_B200_EINVAL;
    if (bnd_slots)
        return loc_pir_program_impl(Q, R, l, m, x_slots, y_slots, bnd_slots, svc_slots, out_slots,
                                    scratch_first, xor_tree, ops, count, comparator);
    if (comparator == 1 || !count || !Q || !R || l < 2 || l > 63 || !m || !x_slots || !y_slots ||
        !svc_slots || !out_slots || xor_tree < 0 || xor_tree > 2)
        return LOCPIR_B200_EINVAL;
    try {
        std::vector<locpir_b200_gate_op> v;
        emit_loc_pir_folded(v, Q, R, l, m, x_slots, y_slots, boxes, svc_slots, out_slots,
                            scratch_first, xor_tree, comparator == 2);
        if (ops) {
            if (*count < v.size())
                return LOCPIR_B200_EINVAL;
            std::copy(v.begin(), v.end(), ops);
        }
        *count = v.size();
        return LOCPIR_B200_OK;
    } catch (...) {
        return LOCPIR_B200_EINVAL;
    }
}

uint64_t locpir_b200_loc_pir_folded_scratch(uint32_t Q, uint32_t R, uint32_t l, uint32_t m)
{
    return loc_pir_folded_scratch(Q, R, l, m);
}

int locpir_b200_loc_pir_folded_program(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                       const uint32_t* x_slots, const uint32_t* y_slots,
                                       const int64_t* boxes, const uint32_t* svc_slots,
                                       const uint32_t* out_slots, uint64_t scratch_first,
                                       int xor_tree, locpir_b200_gate_op* ops, uint64_t* count)
{
    if (!count || !Q || !R || l < 2 || l > 63 || !m || !x_slots || !y_slots || !boxes ||
        !svc_slots || !out_slots || xor_tree < 0 || xor_tree > 2)
        return LOCPIR_B200_EINVAL;
    try {
        std::vector<locpir_b200_gate_op> v;
        emit_loc_pir_folded(v, Q, R, l, m, x_slots, y_slots, boxes, svc_slots, out_slots,
                            scratch_first, xor_tree);
        if (ops) {
            if (*count < v.size())
                return LOCPIR_B200_EINVAL;
            std::copy(v.begin(), v.end(), ops);
        }
        *count = v.size();
        return LOCPIR_B200_OK;
    } catch (...) {
        return LOCPIR_B200_EINVAL;
    }
}

int locpir_b200_loc_pir(locpir_b200_ctx* c, uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                        const uint32_t* x_slots, const uint32_t* y_slots,
                        const uint32_t* bnd_slots, const uint32_t* svc_slots,
                        uint32_t* out_slots, uint64_t scratch_first, int xor_tree)
{
    return guarded(c, [&] {
        if (!Q || !R || l < 2 || !m || !x_slots || !y_slots || !bnd_slots || !svc_slots ||
            !out_slots || xor_tree < 0 || xor_tree > 2)
            throw std::invalid_argument("loc_pir: bad arguments");
        if (scratch_first + loc_pir_scratch(Q, R, l, m) > c->pool_slots)
            throw std::invalid_argument("loc_pir: pool too small for the circuit's scratch");
        std::vector<locpir_b200_gate_op> v;
        emit_loc_pir(v, Q, R, l, m, x_slots, y_slots, bnd_slots, svc_slots, out_slots,
                     scratch_first, xor_tree);
        CK(cudaSetDevice(c->device));
        execute(c, v.data(), v.size());
    });
}

int locpir_b200_check_query_payload(const locpir_b200_params* p, const uint8_t* payload,
                                    uint64_t len, uint32_t l, char* err, uint64_t err_len)
{
    try {
        if (!p || (len && !payload) || l < 2 || l > 255)
            throw std::invalid_argument("bad arguments");
        check_query(p->n, payload, len, l);
        return LOCPIR_B200_OK;
    } catch (const std::exception& e) {
        if (err && err_len) {
            std::snprintf(err, err_len, "%s", e.what());
        }
        return LOCPIR_B200_EINVAL;
    }
}

int locpir_b200_pool_load_queries(locpir_b200_ctx* c, const uint8_t* payloads,
                                  const uint64_t* offsets, uint64_t count, uint32_t l,
                                  const uint32_t* x_first, const uint32_t* y_first)
{
    return guarded(c, [&] {
        if (!count)
            return;
        if (!payloads || !offsets || !x_first || !y_first || l < 2 || l > 255)
            throw std::invalid_argument("pool_load_queries: bad arguments");
        for (uint64_t q = 0; q < count; q++) {
            if (offsets[q + 1] < offsets[q])
                throw std::invalid_argument("pool_load_queries: offsets not ascending");
            check_query(c->p.n, payloads + offsets[q], offsets[q + 1] - offsets[q], l);
            check_pool(c, x_first[q], l);
            check_pool(c, y_first[q], l);
        }
        CK(cudaSetDevice(c->device));
        const uint64_t base = offsets[0], bytes = offsets[count] - base;
        c->h2d_stage.reserve((bytes + 3) / 4, c->stream, false);
        std::vector<uint64_t> offs(offsets, offsets + count + 1);
        for (auto& o : offs)
            o -= base;
        DevBuf<uint64_t> d_off;
        DevBuf<uint32_t> d_slots;
        d_off.reserve(count + 1, c->stream, false);
        d_slots.reserve(2 * count, c->stream, false);
        std::vector<uint32_t> slots(x_first, x_first + count);
        slots.insert(slots.end(), y_first, y_first + count);
        CK(cudaMemcpyAsync(c->h2d_stage.p, payloads + base, bytes, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(d_off.p, offs.data(), (count + 1) * 8, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(d_slots.p, slots.data(), 2 * count * 4, cudaMemcpyHostToDevice, c->stream));
        k_unpack_queries<<<c->num_sms * 4, 256, 0, c->stream>>>(
            dparams(c), reinterpret_cast<const uint8_t*>(c->h2d_stage.p), d_off.p, d_slots.p,
            d_slots.p + count, count, l, c->pool_n.p);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));  // host vectors and temporaries go out of scope
    });
}

int locpir_b200_pool_load_zero_sheet(locpir_b200_ctx* c, const uint8_t* payload, uint64_t len,
                                     uint32_t regions, uint32_t bits,
                                     const uint64_t* service_values, uint32_t svc_first)
{
    return guarded(c, [&] {
        const uint64_t S = 4ull * (c->p.n + 1);
        const uint64_t want = (uint64_t)regions * bits * S;
        if (len != want)  // ZeroSampleSheet::from_payload (circuits.hpp:91-100)
            throw std::invalid_argument("zero-sample sheet payload is " + std::to_string(len) +
                                        " bytes, expected " + std::to_string(want));
        if (!regions || !bits)
            return;
        if (!payload || !service_values)
            throw std::invalid_argument("pool_load_zero_sheet: bad arguments");
        if (bits >= 64)  // preprocess_services (circuits.hpp:125-126)
            throw std::invalid_argument("service bit-length out of range");
        for (uint32_t r = 0; r < regions; r++)
            if (service_values[r] >> bits)
                throw std::invalid_argument("service value " + std::to_string(service_values[r]) +
                                            " does not fit in " + std::to_string(bits) + " bits");
        check_pool(c, svc_first, (uint64_t)regions * bits);
        CK(cudaSetDevice(c->device));
        c->h2d_stage.reserve(len / 4, c->stream, false);
        DevBuf<uint64_t> d_val;
        d_val.reserve(regions, c->stream, false);
        CK(cudaMemcpyAsync(c->h2d_stage.p, payload, len, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(d_val.p, service_values, regions * 8ull, cudaMemcpyHostToDevice, c->stream));
        k_load_zero_sheet<<<c->num_sms * 4, 256, 0, c->stream>>>(dparams(c), c->h2d_stage.p, d_val.p, bits,
                                                               regions, svc_first, c->pool_n.p);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));
    });
}

int locpir_b200_pool_store_responses(locpir_b200_ctx* c, const uint32_t* out_first,
                                     uint64_t count, uint32_t m, uint8_t* payloads)
{
    return guarded(c, [&] {
        if (!count || !m)
            return;
        if (!out_first || !payloads)
            throw std::invalid_argument("pool_store_responses: bad arguments");
        for (uint64_t q = 0; q < count; q++)
            check_pool(c, out_first[q], m);
        CK(cudaSetDevice(c->device));
        const uint64_t words = count * m * (uint64_t)(c->p.n + 1);
        c->d2h_stage.reserve(words, c->stream, false);
        DevBuf<uint32_t> d_first;
        d_first.reserve(count, c->stream, false);
        CK(cudaMemcpyAsync(d_first.p, out_first, count * 4, cudaMemcpyHostToDevice, c->stream));
        k_pack_responses<<<c->num_sms * 4, 256, 0, c->stream>>>(dparams(c), c->pool_n.p, d_first.p, count,
                                                              m, c->d2h_stage.p);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(payloads, c->d2h_stage.p, words * 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

// ---- cross-session batcher (server.hpp) ---------------------------------------------
// locpir_b200_server_* entry points may touch the slots the server owns
struct ServerScope {
    locpir_b200_ctx* c;
    explicit ServerScope(locpir_b200_server* s) : c(s ? s->ctx : nullptr)
    {
        if (c)
            c->server_calls++;
    }
    ~ServerScope()
    {
        if (c)
            c->server_calls--;
    }
};

int locpir_b200_server_create(locpir_b200_ctx* c, const int64_t* boxes, const uint64_t* services,
                              uint32_t R, uint32_t l, uint32_t m, uint32_t max_sessions,
                              int folded, locpir_b200_server** out)
{
    return locpir_b200_server_create_at(c, 0, boxes, services, R, l, m, max_sessions, folded, out);
}

int locpir_b200_server_create_at(locpir_b200_ctx* c, uint64_t base_slot, const int64_t* boxes,
                                 const uint64_t* services, uint32_t R, uint32_t l, uint32_t m,
                                 uint32_t max_sessions, int folded, locpir_b200_server** out)
{
    if (!c || !boxes || !services || !out || !R || l < 2 || l > 63 || !m || m >= 64 ||
        !max_sessions || base_slot >= 0xFFFFFFF0ull)
        return LOCPIR_B200_EINVAL;
    *out = nullptr;
    if (c->server_base != UINT64_MAX)
        return fail(c, LOCPIR_B200_ELOGIC, "a batching server already owns this context's pool tail");
    auto s = std::make_unique<locpir_b200_server>();
    s->ctx = c;
    s->base = (uint32_t)base_slot;
    s->R = R;
    s->l = l;
    s->m = m;
    s->n = c->p.n;
    s->max_sessions = max_sessions;
    s->folded = folded ? 1 : 0;
    s->boxes.assign(boxes, boxes + (size_t)R * 4);
    s->services.assign(services, services + R);
    c->server_base = base_slot;  // claimed now; released below if creation fails
    ServerScope scope(s.get());
    const int rc = lpb::srv_guard(s.get(), [&] {
        for (int64_t v : s->boxes)
            if (v < -(1ll << (l - 1)) || v >= (1ll << (l - 1)))
                throw std::invalid_argument("box boundary does not fit in l bits");
        for (uint64_t v : s->services)
            if (v >> m)
                throw std::invalid_argument("service value " + std::to_string(v) +
                                            " does not fit in " + std::to_string(m) + " bits");
        lpb::srv_init(s.get());
    });
    if (rc) {
        c->err = s->err;
        c->server_base = UINT64_MAX;
        return rc;
    }
    *out = s.release();
    return LOCPIR_B200_OK;
}

void locpir_b200_server_destroy(locpir_b200_server* s)
{
    if (s && s->ctx)
        s->ctx->server_base = UINT64_MAX;  // the pool tail is free again
    delete s;
}

const char* locpir_b200_server_last_error(const locpir_b200_server* s)
{
    return s ? s->err.c_str() : "";
}

int locpir_b200_server_open_session(locpir_b200_server* s, const uint8_t* zero_sheet, uint64_t len,
                                    uint32_t* session)
{
    ServerScope scope(s);
    return lpb::srv_guard(s, [&] {
        if (!session || (len && !zero_sheet))
            throw std::invalid_argument("open_session: bad arguments");
        *session = lpb::srv_open(s, zero_sheet, len);
    });
}

int locpir_b200_server_close_session(locpir_b200_server* s, uint32_t session)
{
    ServerScope scope(s);
    return lpb::srv_guard(s, [&] {
        if (session >= s->max_sessions || !s->open[session])
            throw std::invalid_argument("unknown session");
        for (const auto& p : s->pending)
            if (p.session == session)
                throw std::logic_error("session has queries pending; flush first");
        s->open[session] = 0;
    });
}

int locpir_b200_server_submit(locpir_b200_server* s, uint32_t session, const uint8_t* query,
                              uint64_t len, uint64_t* ticket)
{
    ServerScope scope(s);
    return lpb::srv_guard(s, [&] {
        if (!ticket || (len && !query))
            throw std::invalid_argument("submit: bad arguments");
        *ticket = lpb::srv_submit(s, session, query, len);
    });
}

uint64_t locpir_b200_server_pending(const locpir_b200_server* s) { return s ? s->pending.size() : 0; }

int locpir_b200_server_flush(locpir_b200_server* s, uint64_t* answered)
{
    ServerScope scope(s);
    return lpb::srv_guard(s, [&] {
        const uint64_t n = lpb::srv_flush(s);
        if (answered)
            *answered = n;
    });
}

int locpir_b200_server_take_response(locpir_b200_server* s, uint64_t ticket, uint8_t* out,
                                     uint64_t len)
{
    return lpb::srv_guard(s, [&] {
        auto it = s->responses.find(ticket);
        if (it == s->responses.end())
            throw std::logic_error("ticket " + std::to_string(ticket) + " has no response (not flushed)");
        if (!out || len != it->second.size())
            throw std::invalid_argument("response buffer must be " + std::to_string(it->second.size()) +
                                        " bytes");
        std::memcpy(out, it->second.data(), len);
        s->responses.erase(it);
    });
}

int locpir_b200_client_encrypt(locpir_b200_ctx* c, const uint8_t* lwe_key, uint64_t seed,
                               uint32_t first_index, const uint32_t* mus, uint64_t count,
                               uint64_t first_slot)
{
    return guarded(c, [&] {
        if (!count)
            return;
        if (!lwe_key || !mus)
            throw std::invalid_argument("client_encrypt: bad arguments");
        if ((uint64_t)first_index + count > (1ull << 32))
            throw std::invalid_argument("client_encrypt: stream index range exceeds 2^32");
        for (uint32_t i = 0; i < c->p.n; i++)
            if (lwe_key[i] > 1)
                throw std::invalid_argument("client_encrypt: key bits must be 0 or 1");
        check_pool(c, first_slot, count);
        CK(cudaSetDevice(c->device));
        DevBuf<uint8_t> d_key;
        DevBuf<uint32_t> d_mu;
        d_key.reserve(c->p.n, c->stream, false);
        d_mu.reserve(count, c->stream, false);
        CK(cudaMemcpyAsync(d_key.p, lwe_key, c->p.n, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(d_mu.p, mus, count * 4, cudaMemcpyHostToDevice, c->stream));
        const uint64_t blocks = std::min<uint64_t>((count + 7) / 8, (uint64_t)c->num_sms * 16);
        k_client_encrypt<<<(unsigned)blocks, 256, 0, c->stream>>>(dparams(c), d_key.p, seed, first_index,
                                                                d_mu.p, count, c->p.alpha_in,
                                                                first_slot, c->pool_n.p);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(c->stream));
    });
}

int locpir_b200_debug_fft_error(locpir_b200_ctx* c, const uint32_t* lwe_n, uint64_t count,
                                double* max_err)
{
    return guarded(c, [&] {
        if (!max_err || (count && !lwe_n))
            throw std::invalid_argument("null buffer");
        need_keys(c);
        CK(cudaSetDevice(c->device));
        *max_err = 0.0;
        if (!count)
            return;
        if (c->pool_slots < count) {
            int rc = locpir_b200_pool_reserve(c, count);
            if (rc)
                throw CudaError(c->err);
        }
        pool_copy(c, 0, count, lwe_n, nullptr, cudaMemcpyHostToDevice, true);
        std::vector<BrItem> items(count);
        for (uint64_t g = 0; g < count; g++)
            items[g] = {(uint32_t)g, SLOT_NONE, 1, 0, 0u, (uint32_t)g, SLOT_NONE, 0};
        if (count > c->scratch_slots) {
            grow_scratch(c, count);
            c->scratch_slots = c->pool_N.n / c->dp.N_stride;
        }
        DevBuf<BrItem> d;
        DevBuf<unsigned long long> e;
        d.reserve(count + 1, c->stream, false);
        e.reserve(1, c->stream, false);
        CK(cudaMemsetAsync(e.p, 0, sizeof(unsigned long long), c->stream));
        CK(cudaMemcpyAsync(d.p, items.data(), count * sizeof(BrItem), cudaMemcpyHostToDevice, c->stream));
        const uint32_t mu = 0x20000000u;
        if (c->p.bk_l == 3 && c->p.bk_bgbit == 7)
            k_blind_rotate<3, 7, true><<<(unsigned)count, 64, 0, c->stream>>>(
                dparams(c), d.p, c->pool_n.p, c->pool_N.p, c->bkf.p, tabs(c), mu, e.p);
        else if (c->p.bk_l == 2 && c->p.bk_bgbit == 10)
            k_blind_rotate<2, 10, true><<<(unsigned)count, 64, 0, c->stream>>>(
                dparams(c), d.p, c->pool_n.p, c->pool_N.p, c->bkf.p, tabs(c), mu, e.p);
        else
            throw std::invalid_argument("no blind-rotate kernel instantiated for this (l, Bgbit)");
        CK(cudaGetLastError());
        unsigned long long bits = 0;
        CK(cudaMemcpyAsync(&bits, e.p, sizeof bits, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        std::memcpy(max_err, &bits, sizeof bits);
    });
}

int locpir_b200_timing_enable(locpir_b200_ctx* c, int on)
{
    if (!c)
        return LOCPIR_B200_EINVAL;
    c->timing = on != 0;
    return LOCPIR_B200_OK;
}

int locpir_b200_kernel_stats(locpir_b200_ctx* c, double ms[3], uint64_t launches[3])
{
    return guarded(c, [&] {
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
        for (int k = 0; k < 3; k++) {
            auto& v = c->timer.ev[k];
            for (size_t i = 0; i + 1 < v.size(); i += 2) {
                float t = 0;
                CK(cudaEventElapsedTime(&t, v[i], v[i + 1]));
                c->timer.ms[k] += t;
            }
            for (auto e : v)
                cudaEventDestroy(e);
            v.clear();
            if (ms)
                ms[k] = c->timer.ms[k];
            if (launches)
                launches[k] = c->timer.launches[k];
            c->timer.ms[k] = 0;
            c->timer.launches[k] = 0;
        }
    });
}

int locpir_b200_fp64_peak(locpir_b200_ctx* c, double* tflops)
{
    return guarded(c, [&] {
        if (!tflops)
            throw std::invalid_argument("null output");
        CK(cudaSetDevice(c->device));
        DevBuf<double> sink;
        sink.reserve(1, c->stream, false);
        const int iters = 1 << 16, threads = 256, blocks = c->num_sms * 8;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        k_fp64_peak<<<blocks, threads, 0, c->stream>>>(sink.p, 256);  // warm-up
        double best = 0;
        for (int rep = 0; rep < 3; rep++) {
            CK(cudaEventRecord(e0, c->stream));
            k_fp64_peak<<<blocks, threads, 0, c->stream>>>(sink.p, iters);
            CK(cudaEventRecord(e1, c->stream));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double flops = 2.0 * 8.0 * iters * (double)threads * blocks;
            best = std::max(best, flops / (ms * 1e-3) / 1e12);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *tflops = best;
    });
}

}  // extern "C"
