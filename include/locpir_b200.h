/*
 * locpir_b200.h -- C ABI of the B200-native TFHE gate-bootstrapping engine for
 * LocPIR (arxiv 2407.19871).
 *
 * Drop-in boundary.  The reference's engine boundary is the header-only C++
 * class locpir::GateEngine (/root/reference/proj/include/locpir/gate_engine.hpp:
 * 130-336); its bootstrap step is the secret-key stand-in bootstrap_oracle
 * (gate_engine.hpp:117-123) which the reference names as the plug-in point
 * for a production backend (gate_engine.hpp:113-114).  This ABI exports that
 * backend: plain pointers and sizes, integer status codes, no exceptions and no
 * torch types.  The C++ mirror of GateEngine (paper_2407_19871_b200/host/
 * locpir_b200.hpp) and the Python ctypes mirror (paper_2407_19871_b200/) map
 * the status codes back to the reference's exception types:
 *   LOCPIR_B200_EINVAL -> std::invalid_argument   (gate_engine.hpp:310-320)
 *   LOCPIR_B200_ELOGIC -> std::logic_error        (gate_engine.hpp:304-308)
 *
 * Layouts.  An LWE sample is n+1 little-endian u32 words, mask then body --
 * exactly the reference wire layout (torus.hpp:226-237).  Host buffers are
 * [count][n+1]; device slots are padded to a 16-byte multiple internally.
 * Threading: one context per GPU; a context (and a server built on it) is not
 * thread-safe (as a GateEngine, gate_engine.hpp:335).  Execution is deterministic:
 * the only device randomness, locpir_b200_client_encrypt, is a counter-based stream
 * (a pure function of key, seed and stream index).
 */
#ifndef LOCPIR_B200_H
#define LOCPIR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOCPIR_B200_OK 0
#define LOCPIR_B200_EINVAL (-1)
#define LOCPIR_B200_ELOGIC (-2)
#define LOCPIR_B200_ECUDA (-3)
#define LOCPIR_B200_ENOMEM (-4)

/* Gate kinds.  AND/OR/XOR/XNOR/NOT/MUX are the reference's gate set
 * (gate_engine.hpp:196-269); NAND/NOR are the TFHE forms BASELINE.json cfg2 needs. */
#define LOCPIR_B200_AND 0
#define LOCPIR_B200_OR 1
#define LOCPIR_B200_XOR 2
#define LOCPIR_B200_XNOR 3
#define LOCPIR_B200_NAND 4
#define LOCPIR_B200_MUX 5  /* out = in0 ? in1 : in2 */
#define LOCPIR_B200_NOT 6  /* free: componentwise negation (gate_engine.hpp:243-250) */
#define LOCPIR_B200_NOR 7
#define LOCPIR_B200_COPY 8 /* free: out = in0 */
#define LOCPIR_B200_CONST 9 /* free: out = trivial sample encode_bit(in0 != 0) (gate_engine.hpp:174-179) */
#define LOCPIR_B200_ANDNY 10 /* AND(NOT in0, in1): one bootstrap, form (-1/8, -1, +1) */
#define LOCPIR_B200_ORNY 11  /* OR(NOT in0, in1):  one bootstrap, form (+1/8, -1, +1) */
#define LOCPIR_B200_MAJ 12   /* MAJ(in0, in1, in2): one bootstrap of in0 + in1 + in2 (three
                                +-1/8 never sum to 0); counted in bootstrap_units */
#define LOCPIR_B200_XOR3 13  /* in0 ^ in1 ^ in2: one bootstrap of -2 (in0 + in1 + in2) -- an
                                odd count of true inputs lands on +1/4, an even count on
                                -1/4 (mod 1), the margins of the 2-input XOR; flagged
                                modes' ternary XOR trees; counted in bootstrap_units */

/* Full TFHE parameter set (extends TlweParams {n, sigma}, torus.hpp:71-110). */
typedef struct locpir_b200_params {
    uint32_t n;       /* LWE dimension */
    uint32_t N;       /* TRLWE ring degree (power of two, 1024) */
    uint32_t k;       /* TRLWE rank (1) */
    uint32_t bk_l;    /* BK gadget length */
    uint32_t bk_bgbit;/* log2 of BK gadget base */
    uint32_t ks_t;    /* key-switch length */
    uint32_t ks_basebit;
    double alpha_in;  /* LWE / key-switch noise stddev (torus fraction) */
    double alpha_bk;  /* bootstrapping-key noise stddev */
} locpir_b200_params;

/* One gate of a program.  Operands index n-dim slots of the context's device pool;
 * unused operands are LOCPIR_B200_NONE_SLOT (CONST carries its bit in in0). */
#define LOCPIR_B200_NONE_SLOT 0xFFFFFFFFu
typedef struct locpir_b200_gate_op {
    uint32_t kind;
    uint32_t in0, in1, in2;
    uint32_t out;
} locpir_b200_gate_op;

typedef struct locpir_b200_ctx locpir_b200_ctx;

/* ---- parameters (host only) ---------------------------------------------- */
/* security_bits = 80 (BASELINE configs[0]) or 128 (configs[1]) */
int locpir_b200_params_default(int security_bits, locpir_b200_params* out);
size_t locpir_b200_bk_words(const locpir_b200_params* p);  /* torus-form BK words */
size_t locpir_b200_ksk_words(const locpir_b200_params* p); /* KSK words [N][t][base-1][n+1] */

/* ---- client-side key material and encryption (host only, no GPU) ----------
 * Replaces keygen (torus.hpp:146-154), extended with the TRLWE key, BK and KSK.
 * All randomness is the reference NoiseSampler (mt19937_64 + normal_distribution,
 * torus.hpp:119-138).  Any output pointer may be NULL to skip it. */
int locpir_b200_keygen(const locpir_b200_params* p, uint64_t seed, uint8_t* lwe_key,
                       uint8_t* trlwe_key, uint32_t* bk, uint32_t* ksk);
/* The same derivation around a caller's LWE key (n bytes, 0/1), e.g. a reference
 * SecretKey from keygen(params, key_seed) (torus.hpp:146-154): the TRLWE key, BK and KSK
 * come from `seed` exactly as in locpir_b200_keygen, which this equals when
 * lwe_key == keygen(n, seed). */
int locpir_b200_keygen_with_lwe_key(const locpir_b200_params* p, uint64_t seed,
                                    const uint8_t* lwe_key, uint8_t* trlwe_key, uint32_t* bk,
                                    uint32_t* ksk);
/* encrypt_bit (torus.hpp:172-175) of bits[i] with NoiseSampler(seed, alpha_in),
 * drawn in order i = 0..count-1; out is [count][n+1]. */
int locpir_b200_encrypt_bits(const locpir_b200_params* p, const uint8_t* lwe_key, uint64_t seed,
                             const uint8_t* bits, uint64_t count, uint32_t* out);
/* decrypt_bit (torus.hpp:191-194) */
int locpir_b200_decrypt_bits(const locpir_b200_params* p, const uint8_t* lwe_key,
                             const uint32_t* cts, uint64_t count, uint8_t* bits_out);

/* ---- device context -------------------------------------------------------- */
/* stream: a cudaStream_t to launch on, or NULL for a context-owned stream. */
int locpir_b200_ctx_create(const locpir_b200_params* p, int device, void* stream,
                           locpir_b200_ctx** out);
void locpir_b200_ctx_destroy(locpir_b200_ctx* ctx);
const char* locpir_b200_last_error(const locpir_b200_ctx* ctx);
void* locpir_b200_stream(const locpir_b200_ctx* ctx);

/* Bootstrapping key (torus form [n][(k+1)l][k+1][N]) and key-switching key
 * ([N][t][base-1][n+1]).  on_device != 0: the pointers are device memory (e.g.
 * received by an NCCL broadcast).  The BK is transformed to the frequency domain
 * on the device (kernel K0). */
int locpir_b200_upload_keys(locpir_b200_ctx* ctx, const uint32_t* bk, const uint32_t* ksk,
                            int on_device);

/* ---- device ciphertext pool --------------------------------------------------- */
int locpir_b200_pool_reserve(locpir_b200_ctx* ctx, uint64_t slots);
uint64_t locpir_b200_pool_capacity(const locpir_b200_ctx* ctx);
int locpir_b200_pool_h2d(locpir_b200_ctx* ctx, uint64_t first, uint64_t count,
                         const uint32_t* host);
int locpir_b200_pool_d2h(locpir_b200_ctx* ctx, uint64_t first, uint64_t count, uint32_t* host);
/* device-to-device copy into the pool from a [count][n+1] device buffer */
int locpir_b200_pool_load_device(locpir_b200_ctx* ctx, uint64_t first, uint64_t count,
                                 const uint32_t* dev);
int locpir_b200_pool_store_device(locpir_b200_ctx* ctx, uint64_t first, uint64_t count,
                                  uint32_t* dev);

/* ---- gate programs ------------------------------------------------------------
 * Runs ops in program order semantics; the circuit scheduler assigns every gate
 * to the earliest depth level its inputs allow, splits MUX into its two blind
 * rotations (the "else" half leaves the critical path), and launches each level
 * as one batched blind-rotate kernel plus one batched key-switch kernel.
 * Each op's out slot must not be read by an earlier op of the same program. */
int locpir_b200_run(locpir_b200_ctx* ctx, const locpir_b200_gate_op* ops, uint64_t count);
/* SURVEY §8(b) contract name: evaluate one level of mutually independent gates. */
int locpir_b200_eval_level(locpir_b200_ctx* ctx, const locpir_b200_gate_op* ops,
                           uint64_t count);
int locpir_b200_sync(locpir_b200_ctx* ctx);

/* Pre-planned program: the schedule and the per-level work lists are built and
 * uploaded once; program_launch only enqueues the level kernels on the context
 * stream (asynchronous; no host work, graph-capturable). */
typedef struct locpir_b200_program locpir_b200_program;
int locpir_b200_program_create(locpir_b200_ctx* ctx, const locpir_b200_gate_op* ops,
                               uint64_t count, locpir_b200_program** out);
int locpir_b200_program_launch(locpir_b200_ctx* ctx, locpir_b200_program* prog);
/* Sizes the context's scratch for the program (and checks the keys are uploaded) so
 * that its first launch allocates nothing; optional. */
int locpir_b200_program_prepare(locpir_b200_ctx* ctx, locpir_b200_program* prog);
/* kernel launches one program_launch issues */
uint64_t locpir_b200_program_kernels(const locpir_b200_program* prog);
void locpir_b200_program_destroy(locpir_b200_program* prog);

/* Host-only plan of a program (no GPU): number of bootstrap levels, blind rotations,
 * key switches; used by tests and the C++ mirror. */
int locpir_b200_plan(const locpir_b200_gate_op* ops, uint64_t count, uint32_t* levels,
                     uint64_t* blind_rotations, uint64_t* key_switches);

/* Counters (gate_engine.hpp:31-77): and, or, xor, xnor, not, mux, nand, nor,
 * bootstrap_units (= and+or+xor+xnor+nand+nor+2*mux). */
int locpir_b200_counters(const locpir_b200_ctx* ctx, uint64_t out[9]);
int locpir_b200_counters_reset(locpir_b200_ctx* ctx);

/* ---- end-to-end convenience: one batched gate on HOST buffers ------------------
 * out[i] = gate(a[i], b[i]) for i < count; a, b, out are [count][n+1] host arrays.
 * Includes the host->device and device->host transfers.  When a and b are pinned
 * (device-mapped, e.g. cudaHostAlloc) and count >= 256, the blind rotation reads the
 * input rows over PCIe itself (zero-copy; LOCPIR_B200_ZEROCOPY=0 at context creation
 * disables it); otherwise they are copied first.  Results are identical either way.
 * The context's pool slots [0, count) (zero-copy) or [0, 3 count) (copy) are used. */
int locpir_b200_gate_batch_host(locpir_b200_ctx* ctx, uint32_t kind, const uint32_t* a,
                                const uint32_t* b, uint32_t* out, uint64_t count);

/* ---- circuits (circuits.hpp:187-324), batched over queries ---------------------
 * loc_pir for Q independent queries against R regions:
 *   x_slots, y_slots : [Q][l] pool slots of the query words (LSB first)
 *   bnd_slots        : [R][4][l] pool slots of x1, x2, y1, y2 (circuits.hpp:22-27)
 *   svc_slots        : [R][m] pool slots of the service bits
 *   out_slots        : [Q][m] pool slots receiving the XOR-sum result
 *   scratch_first    : first pool slot the circuit may use for intermediates
 *                      (needs locpir_b200_loc_pir_scratch() slots)
 *   xor_tree         : 0 = the reference's N-long XOR chain (circuits.hpp:257-261),
 *                      1 = balanced tree (same N*m XOR count, log2 N depth),
 *                      2 = box-sharded partial: tree root copied to out_slots without
 *                          the final XOR with Enc(0) (N-1 XORs per column); a rank-0
 *                          combine of the shards' partials restores N*m.
 * Gate counts follow N(12l + 2m + 3) units per query (bench.hpp:35-43). */
uint64_t locpir_b200_loc_pir_scratch(uint32_t Q, uint32_t R, uint32_t l, uint32_t m);
int locpir_b200_loc_pir(locpir_b200_ctx* ctx, uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                        const uint32_t* x_slots, const uint32_t* y_slots,
                        const uint32_t* bnd_slots, const uint32_t* svc_slots,
                        uint32_t* out_slots, uint64_t scratch_first, int xor_tree);
/* Emit the loc_pir gate program without running it (host only). */
int locpir_b200_loc_pir_program(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                const uint32_t* x_slots, const uint32_t* y_slots,
                                const uint32_t* bnd_slots, const uint32_t* svc_slots,
                                const uint32_t* out_slots, uint64_t scratch_first,
                                int xor_tree, locpir_b200_gate_op* ops, uint64_t* count);

/* ---- stage-wise parity hooks (diagnostics; host buffers, synchronous) -----------
 * blind rotation + sample extraction of one combined LWE (n+1 words, the gate's
 * linear form already applied) -> N-dim LWE (N+1 words): the pre-key-switch
 * coefficients the parity ladder compares with the exact oracle. */
int locpir_b200_debug_blind_rotate(locpir_b200_ctx* ctx, const uint32_t* lwe_n, uint64_t count,
                                   uint32_t* out_N);
/* key switch of N-dim LWEs (N+1 words each) -> n-dim (n+1 words each) */
/* FFT rounding margin: blind-rotates count combined n-dim LWEs with a diagnostic build of
 * the throughput kernel and returns max |w - rint(w)| over every inverse-transform output
 * before rounding (the pre-KS coefficients are exact iff this stays below 1/2). */
int locpir_b200_debug_fft_error(locpir_b200_ctx* ctx, const uint32_t* lwe_n, uint64_t count,
                                double* max_err);
int locpir_b200_debug_keyswitch(locpir_b200_ctx* ctx, const uint32_t* lwe_N, uint64_t count,
                                uint32_t* out_n);

/* ---- wire payloads <-> device pool --------------------------------
 * The reference's session payloads go to and from the pool without a host-side
 * per-sample pass: one 1-D copy of the bytes plus an unpack/pack kernel.
 *   QUERY    (protocol.hpp:185-193): two framed words, each u8 length l then l raw
 *            samples (codec.hpp:172-193) -- the prefix leaves the second word
 *            misaligned, so the kernel assembles words from bytes.
 *   ZEROSHEET (circuits.hpp:46-54, :83-104): regions*bits raw zero samples; loading it
 *            also applies preprocess_services (circuits.hpp:118-146): sample + trivial
 *            encode_bit(service bit), region-major, bit-minor.
 *   RESPONSE (protocol.hpp:212-227): m raw samples per query.
 * Validation mirrors the reference's DecodeError / out_of_range checks (EINVAL with the
 * reference's message). */
/* Host-only framing check of one QUERY payload (no GPU needed); err may be NULL. */
int locpir_b200_check_query_payload(const locpir_b200_params* p, const uint8_t* payload,
                                    uint64_t len, uint32_t l, char* err, uint64_t err_len);
/* count QUERY payloads concatenated; payload q = bytes [offsets[q], offsets[q+1]).
 * Word bits i go to slots x_first[q] + i and y_first[q] + i (LSB first). */
int locpir_b200_pool_load_queries(locpir_b200_ctx* c, const uint8_t* payloads,
                                  const uint64_t* offsets, uint64_t count, uint32_t l,
                                  const uint32_t* x_first, const uint32_t* y_first);
/* One ZEROSHEET payload + the server's service values -> encrypted service bits at
 * slots svc_first + r*bits + j. */
int locpir_b200_pool_load_zero_sheet(locpir_b200_ctx* c, const uint8_t* payload, uint64_t len,
                                     uint32_t regions, uint32_t bits,
                                     const uint64_t* service_values, uint32_t svc_first);
/* RESPONSE payloads of count queries (m samples from slot out_first[q] on), written
 * back to back into payloads (count * m * 4(n+1) bytes). */
int locpir_b200_pool_store_responses(locpir_b200_ctx* c, const uint32_t* out_first,
                                     uint64_t count, uint32_t m, uint8_t* payloads);

/* ---- cross-session query batcher -----------------------------------
 * Server::handle_zerosheet / handle_query (protocol.hpp:373-424) without the transport:
 * sessions register their ZEROSHEET once, QUERY payloads from any session queue up, and
 * flush() answers all of them with ONE level-scheduled program (each query reads its own
 * session's preprocessed services), producing RESPONSE payloads per ticket.  boxes: [R][4]
 * signed l-bit grid values (x1, x2, y1, y2) of the server's dataset; services: [R] values.
 * folded = 1 uses the plaintext-boundary constant-folded circuit (flagged mode). */
typedef struct locpir_b200_server locpir_b200_server;
int locpir_b200_server_create(locpir_b200_ctx* c, const int64_t* boxes, const uint64_t* services,
                              uint32_t R, uint32_t l, uint32_t m, uint32_t max_sessions,
                              int folded, locpir_b200_server** out);
/* The server owns every pool slot from base_slot on (server_create: base_slot = 0, i.e. a
 * dedicated context).  While it exists, any other call on the context that reads or
 * writes one of those slots fails with EINVAL -- e.g. a GateEngine sharing the context
 * must keep its slots below base_slot.  One server per context; destroy the server
 * before its context. */
int locpir_b200_server_create_at(locpir_b200_ctx* c, uint64_t base_slot, const int64_t* boxes,
                                 const uint64_t* services, uint32_t R, uint32_t l, uint32_t m,
                                 uint32_t max_sessions, int folded, locpir_b200_server** out);
void locpir_b200_server_destroy(locpir_b200_server* s);
const char* locpir_b200_server_last_error(const locpir_b200_server* s);
int locpir_b200_server_open_session(locpir_b200_server* s, const uint8_t* zero_sheet, uint64_t len,
                                    uint32_t* session);
int locpir_b200_server_close_session(locpir_b200_server* s, uint32_t session);
int locpir_b200_server_submit(locpir_b200_server* s, uint32_t session, const uint8_t* query,
                              uint64_t len, uint64_t* ticket);
uint64_t locpir_b200_server_pending(const locpir_b200_server* s);
int locpir_b200_server_flush(locpir_b200_server* s, uint64_t* answered);
/* RESPONSE payload of a flushed ticket (m * 4(n+1) bytes); ELOGIC if not answered yet. */
int locpir_b200_server_take_response(locpir_b200_server* s, uint64_t ticket, uint8_t* out,
                                     uint64_t len);

/* ---- client-side batched encryption on the device --------------------
 * Encrypts torus messages mus[j] under the client's LWE key (n bytes, 0/1) into pool
 * slots first_slot + j, with the counter-based stream of csrc/cbrng.h (Philox4x32-10 +
 * IEEE-exact Box-Muller, noise alpha_in): sample j uses stream index first_index + j, so
 * the output is a pure function of (key, seed, index, mu) and equals the CPU definition
 * bit for bit.  mu = +-1/8 encrypts bits (torus.hpp:52-55, :172-175); mu = 0 makes the
 * zero-sample sheet (circuits.hpp:46-54).  Flagged mode: not the reference's mt19937_64
 * stream (torus.hpp:119-138). */
int locpir_b200_client_encrypt(locpir_b200_ctx* c, const uint8_t* lwe_key, uint64_t seed,
                               uint32_t first_index, const uint32_t* mus, uint64_t count,
                               uint64_t first_slot);

/* ---- flagged mode: plaintext-boundary constant folding -------------
 * The server's box boundaries are plaintext (dataset.hpp:250-253).  Comparing an
 * encrypted word against a known word folds every XNOR into a free (or no) negation and
 * every MUX into one AND/OR-with-negated-input bootstrap, and the first bit into a free
 * gate: about 4l + 2m per region instead of 12l + 2m + 3 (the reference count model no
 * longer applies -- hence a separate entry point).  boxes: [R][4] signed grid values
 * (x1, x2, y1, y2) of l-bit two's-complement words; results decrypt identically. */
uint64_t locpir_b200_loc_pir_folded_scratch(uint32_t Q, uint32_t R, uint32_t l, uint32_t m);
/* Flagged mode: comparators as a majority borrow chain (works with ENCRYPTED boundaries,
 * cfg5): with the sign bits flipped, a < b = borrow out of a - b,
 * borrow_{i+1} = MAJ(NOT a_i, b_i, borrow_i), borrow_0 = 0 -- l bootstraps per comparator
 * instead of 3l, same depth; a region costs 4l + 2m + 3, minus m per query: like every
 * flagged mode it skips the bootstrapped XOR with Enc(0) that starts each bit column of
 * the reference's XOR sum (one circuit level).  Same arguments as
 * locpir_b200_loc_pir_program; decrypted results equal the reference circuit's. */
int locpir_b200_loc_pir_maj_program(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                    const uint32_t* x_slots, const uint32_t* y_slots,
                                    const uint32_t* bnd_slots, const uint32_t* svc_slots,
                                    const uint32_t* out_slots, uint64_t scratch_first,
                                    int xor_tree, locpir_b200_gate_op* ops, uint64_t* count);
/* General emitter.  Exactly one of bnd_slots ([R][4][l] pool slots, as
 * locpir_b200_loc_pir_program) or boxes ([R][4] plaintext signed grid values, folded as
 * locpir_b200_loc_pir_folded_program) is non-NULL.  comparator: 0 = reference XNOR/MUX
 * chain (folded chain for plaintext boxes), 1 = majority borrow chain (slots only),
 * 2 = log-depth tree (flagged latency mode: depth log2 l, +1 with encrypted boundaries,
 * more gates; for latency-bound batches such as cfg1).  Scratch: locpir_b200_loc_pir_scratch
 * bounds every mode. */
int locpir_b200_loc_pir_program_ex(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                   const uint32_t* x_slots, const uint32_t* y_slots,
                                   const uint32_t* bnd_slots, const int64_t* boxes,
                                   const uint32_t* svc_slots, const uint32_t* out_slots,
                                   uint64_t scratch_first, int xor_tree, int comparator,
                                   locpir_b200_gate_op* ops, uint64_t* count);
int locpir_b200_loc_pir_folded_program(uint32_t Q, uint32_t R, uint32_t l, uint32_t m,
                                       const uint32_t* x_slots, const uint32_t* y_slots,
                                       const int64_t* boxes, const uint32_t* svc_slots,
                                       const uint32_t* out_slots, uint64_t scratch_first,
                                       int xor_tree, locpir_b200_gate_op* ops, uint64_t* count);

/* ---- instrumentation -------------------------------------------------------------
 * Per-kernel device time (CUDA events on the context stream) accumulated since the
 * last reset: [0] blind-rotate ms, [1] key-switch ms, [2] linear ms; launches in
 * launches[0..2].  Timing is off unless enabled (it adds event records). */
int locpir_b200_timing_enable(locpir_b200_ctx* ctx, int on);
int locpir_b200_kernel_stats(locpir_b200_ctx* ctx, double ms[3], uint64_t launches[3]);
/* FP64 FMA microbenchmark on the context's device: returns achieved TFLOP/s
 * (2 flops per DFMA) -- the measured denominator of the bootstrap roofline. */
int locpir_b200_fp64_peak(locpir_b200_ctx* ctx, double* tflops);

#ifdef __cplusplus
}
#endif
#endif
