"""Python mirror of the reference engine boundary over the B200 C ABI.

Mirrors locpir::GateEngine (/root/reference/proj/include/locpir/gate_engine.hpp:
130-336) -- same method names, argument meaning and error behaviour -- with a
new engine kind "tfhe-b200" (``parse_engine_kind("tfhe")`` keeps throwing, as
test_gate_engine.cpp:154 pins).  Every bootstrapped gate runs on the GPU through
include/locpir_b200.h; there is no CPU path.

Differences the real bootstrap forces:
  * bootstrapping is deterministic, so ``fork(lane)`` shares everything and only
    exists for API compatibility;
  * the stand-in's exact-tie sign rule (phase exactly 0 -> 0) does not apply;
  * gates can be recorded and run level-batched: ``with engine.batch(): ...``.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import itertools
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._abi import GateOp, lib

ENGINE_KINDS = ("clear", "tlwe-oracle", "tfhe-b200")


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference (gate_engine.hpp:310-320, torus.hpp:179-217)."""


class LogicError(RuntimeError):
    """std::logic_error of the reference (gate_engine.hpp:304-308)."""


class CudaError(RuntimeError):
    pass


def parse_engine_kind(s: str) -> str:
    """gate_engine.hpp:21-29 plus the new "tfhe-b200" kind."""
    if s in ENGINE_KINDS:
        return s
    raise InvalidArgument(f'unknown engine "{s}" (expected clear, tlwe-oracle or tfhe-b200)')


def _check(rc: int, ctx=None):
    if rc == _abi.OK:
        return
    msg = lib().locpir_b200_last_error(ctx).decode() if ctx else ""
    if rc == _abi.EINVAL:
        raise InvalidArgument(msg or "invalid argument")
    if rc == _abi.ELOGIC:
        raise LogicError(msg or "logic error")
    if rc == _abi.ENOMEM:
        raise MemoryError(msg)
    raise CudaError(msg or f"CUDA error ({rc})")


def _u32(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


# ---------------------------------------------------------------------------
# parameters and client-side key material
# ---------------------------------------------------------------------------
class TfheParams:
    """Full TFHE parameter set (extends TlweParams, torus.hpp:71-110)."""

    def __init__(self, security_bits: int = 128):
        self.c = _abi.Params()
        _check(lib().locpir_b200_params_default(security_bits, C.byref(self.c)))
        self.security_bits = security_bits

    @classmethod
    def tfhe80(cls):
        return cls(80)

    @classmethod
    def tfhe128(cls):
        return cls(128)

    @property
    def n(self):
        return self.c.n

    @property
    def N(self):
        return self.c.N

    @property
    def sigma(self):
        return self.c.alpha_in

    def sample_bytes(self) -> int:
        return 4 * (self.n + 1)  # torus.hpp:227-230

    def bk_words(self) -> int:
        return lib().locpir_b200_bk_words(C.byref(self.c))

    def ksk_words(self) -> int:
        return lib().locpir_b200_ksk_words(C.byref(self.c))


class ClientKeys:
    """Secret keys plus the public evaluation keys (BK, KSK) from one seed."""

    def __init__(self, params: TfheParams, seed: int, evaluation_keys: bool = True):
        self.params = params
        p = params.c
        self.lwe_key = np.zeros(p.n, np.uint8)
        self.trlwe_key = np.zeros(p.N, np.uint8)
        self.bk = np.zeros(params.bk_words(), np.uint32) if evaluation_keys else None
        self.ksk = np.zeros(params.ksk_words(), np.uint32) if evaluation_keys else None
        _check(lib().locpir_b200_keygen(
            C.byref(p), seed, _u8(self.lwe_key), _u8(self.trlwe_key),
            _u32(self.bk) if evaluation_keys else None,
            _u32(self.ksk) if evaluation_keys else None))

    # ---- key blobs (SURVEY §5 "persist BK/KSK blobs (torus form) to skip keygen") -------
    _MAGIC = b"LOCPIRB200KEYS\x00\x01"

    def save(self, path: str, secret: bool = True):
        """Write the key set to `path`: a header (magic, the 9 parameters), the LWE and
        TRLWE keys (omitted with secret=False: a server-side evaluation-key file), BK and
        KSK in torus form, and a SHA-256 over everything before it."""
        import hashlib
        import struct
        p = self.params.c
        hdr = self._MAGIC + struct.pack("<7I2d?", p.n, p.N, p.k, p.bk_l, p.bk_bgbit, p.ks_t,
                                        p.ks_basebit, p.alpha_in, p.alpha_bk, bool(secret))
        parts = [hdr]
        if secret:
            parts += [self.lwe_key.tobytes(), self.trlwe_key.tobytes()]
        if self.bk is None:
            raise LogicError("no evaluation keys to save")
        parts += [self.bk.astype("<u4").tobytes(), self.ksk.astype("<u4").tobytes()]
        body = b"".join(parts)
        with open(path, "wb") as f:
            f.write(body + hashlib.sha256(body).digest())

    @classmethod
    def load(cls, path: str) -> "ClientKeys":
        """Read a key file written by save(); raises InvalidArgument on a bad magic, an
        unknown parameter set, a truncated file or a checksum mismatch."""
        import hashlib
        import struct
        raw = open(path, "rb").read()
        m = cls._MAGIC
        fmt = "<7I2d?"
        hl = len(m) + struct.calcsize(fmt)
        if len(raw) < hl + 32 or raw[:len(m)] != m:
            raise InvalidArgument(f"{path}: not a locpir_b200 key file")
        body, digest = raw[:-32], raw[-32:]
        if hashlib.sha256(body).digest() != digest:
            raise InvalidArgument(f"{path}: checksum mismatch")
        n, N, k, l, bg, t, bb, ain, abk, secret = struct.unpack(fmt, raw[len(m):hl])
        params = None
        for level in (128, 80):
            q = TfheParams(level)
            c = q.c
            if (c.n, c.N, c.k, c.bk_l, c.bk_bgbit, c.ks_t, c.ks_basebit, c.alpha_in,
                    c.alpha_bk) == (n, N, k, l, bg, t, bb, ain, abk):
                params = q
        if params is None:
            raise InvalidArgument(f"{path}: parameter set is not a BASELINE set")
        keys = cls.__new__(cls)
        keys.params = params
        off = hl
        want = (n + N if secret else 0) + 4 * (params.bk_words() + params.ksk_words())
        if len(body) - hl != want:
            raise InvalidArgument(f"{path}: truncated key file")
        if secret:
            keys.lwe_key = np.frombuffer(body, np.uint8, n, off).copy()
            keys.trlwe_key = np.frombuffer(body, np.uint8, N, off + n).copy()
            off += n + N
        else:
            keys.lwe_key = keys.trlwe_key = None
        keys.bk = np.frombuffer(body, "<u4", params.bk_words(), off).astype(np.uint32)
        off += 4 * params.bk_words()
        keys.ksk = np.frombuffer(body, "<u4", params.ksk_words(), off).astype(np.uint32)
        return keys

    def encrypt_bits(self, bits, seed: int) -> np.ndarray:
        bits = np.ascontiguousarray(np.asarray(bits, np.uint8).reshape(-1))
        out = np.zeros((len(bits), self.params.n + 1), np.uint32)
        _check(lib().locpir_b200_encrypt_bits(C.byref(self.params.c), _u8(self.lwe_key), seed,
                                              _u8(bits), len(bits), _u32(out)))
        return out

    def decrypt_bits(self, cts: np.ndarray) -> np.ndarray:
        cts = np.ascontiguousarray(cts, np.uint32).reshape(-1, self.params.n + 1)
        out = np.zeros(cts.shape[0], np.uint8)
        _check(lib().locpir_b200_decrypt_bits(C.byref(self.params.c), _u8(self.lwe_key),
                                              _u32(cts), cts.shape[0], _u8(out)))
        return out

    def phase(self, ct: np.ndarray) -> int:
        ct = np.asarray(ct, np.uint32)
        n = self.params.n
        return int((int(ct[n]) - int(np.sum(ct[:n].astype(np.uint64) * self.lwe_key))) % 2**32)


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
class Context:
    """One GPU's engine state: keys, ciphertext pool, stream (include/locpir_b200.h)."""

    def __init__(self, params: TfheParams, device: int = 0, stream: int | None = None):
        self.params = params
        h = C.c_void_p()
        _check(lib().locpir_b200_ctx_create(C.byref(params.c), device,
                                            C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().locpir_b200_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:  # interpreter shutdown may already have torn down the module globals
            self.close()
        except Exception:
            pass

    def _c(self, rc):
        _check(rc, self.h)

    @property
    def stream(self) -> int:
        return lib().locpir_b200_stream(self.h) or 0

    def upload_keys(self, bk, ksk, on_device: bool = False):
        """bk/ksk: numpy arrays (host) or integer device pointers (on_device=True)."""
        if on_device:
            self._c(lib().locpir_b200_upload_keys(self.h, C.c_void_p(bk), C.c_void_p(ksk), 1))
        else:
            bk = np.ascontiguousarray(bk, np.uint32)
            ksk = np.ascontiguousarray(ksk, np.uint32)
            self._c(lib().locpir_b200_upload_keys(self.h, bk.ctypes.data, ksk.ctypes.data, 0))

    def pool_reserve(self, slots: int):
        self._c(lib().locpir_b200_pool_reserve(self.h, slots))

    @property
    def pool_capacity(self) -> int:
        return lib().locpir_b200_pool_capacity(self.h)

    def h2d(self, first: int, cts: np.ndarray):
        cts = np.ascontiguousarray(cts, np.uint32).reshape(-1, self.params.n + 1)
        self._c(lib().locpir_b200_pool_h2d(self.h, first, cts.shape[0], cts.ctypes.data))

    def d2h(self, first: int, count: int) -> np.ndarray:
        out = np.zeros((count, self.params.n + 1), np.uint32)
        self._c(lib().locpir_b200_pool_d2h(self.h, first, count, out.ctypes.data))
        return out

    def load_device(self, first: int, count: int, dev_ptr: int):
        self._c(lib().locpir_b200_pool_load_device(self.h, first, count, C.c_void_p(dev_ptr)))

    def store_device(self, first: int, count: int, dev_ptr: int):
        self._c(lib().locpir_b200_pool_store_device(self.h, first, count, C.c_void_p(dev_ptr)))

    @staticmethod
    def ops_array(ops) -> C.Array:
        if isinstance(ops, C.Array):
            return ops
        arr = (GateOp * max(1, len(ops)))()
        for i, (k, a, b, c, o) in enumerate(ops):
            arr[i] = GateOp(k, a, b, c, o)
        return arr

    def run(self, ops):
        """ops: sequence of (kind, in0, in1, in2, out) or a ctypes GateOp array."""
        if not isinstance(ops, C.Array):
            n = len(ops)
            ops = self.ops_array(ops)
        else:
            n = len(ops)
        self._c(lib().locpir_b200_run(self.h, ops, n))

    def program(self, ops) -> "Program":
        """Plan and upload a gate program once; launch() only enqueues kernels."""
        arr = ops if isinstance(ops, C.Array) else self.ops_array(ops)
        h = C.c_void_p()
        self._c(lib().locpir_b200_program_create(self.h, arr, len(arr) if len(ops) else 0,
                                                 C.byref(h)))
        return Program(self, h)

    def eval_level(self, ops):
        arr = self.ops_array(ops)
        self._c(lib().locpir_b200_eval_level(self.h, arr, len(ops)))

    def sync(self):
        self._c(lib().locpir_b200_sync(self.h))

    def counters(self) -> dict:
        a = (C.c_uint64 * 9)()
        self._c(lib().locpir_b200_counters(self.h, a))
        names = ["and", "or", "xor", "xnor", "not", "mux", "nand", "nor", "bootstrap_units"]
        return dict(zip(names, list(a)))

    def counters_reset(self):
        self._c(lib().locpir_b200_counters_reset(self.h))

    def gate_batch_host(self, kind: int, a: np.ndarray, b: np.ndarray,
                        out: np.ndarray | None = None) -> np.ndarray:
        a = np.ascontiguousarray(a, np.uint32)
        b = np.ascontiguousarray(b, np.uint32)
        if out is None:
            out = np.zeros_like(a)
        self._c(lib().locpir_b200_gate_batch_host(self.h, kind, a.ctypes.data, b.ctypes.data,
                                                  out.ctypes.data, a.shape[0]))
        return out

    def gate_batch_host_ptr(self, kind: int, a_ptr: int, b_ptr: int, out_ptr: int, count: int):
        self._c(lib().locpir_b200_gate_batch_host(self.h, kind, C.c_void_p(a_ptr),
                                                  C.c_void_p(b_ptr), C.c_void_p(out_ptr), count))

    def loc_pir(self, Q, R, l, m, x_slots, y_slots, bnd_slots, svc_slots, out_slots,
                scratch_first, xor_tree=True):
        arrs = [np.ascontiguousarray(v, np.uint32).reshape(-1)
                for v in (x_slots, y_slots, bnd_slots, svc_slots, out_slots)]
        self._c(lib().locpir_b200_loc_pir(self.h, Q, R, l, m, *[_u32(v) for v in arrs],
                                          scratch_first, _tree_mode(xor_tree)))

    # -- wire payloads -------------------------------------
    def load_queries(self, payloads, l: int, x_first, y_first):
        """QUERY payloads (protocol.hpp:185-193) -> pool: word bits i at x_first[q] + i and
        y_first[q] + i.  One 1-D copy of all payloads + an unpack kernel."""
        buf = b"".join(payloads)
        offs = np.zeros(len(payloads) + 1, np.uint64)
        offs[1:] = np.cumsum([len(p) for p in payloads])
        xf = np.ascontiguousarray(x_first, np.uint32)
        yf = np.ascontiguousarray(y_first, np.uint32)
        raw = np.frombuffer(buf, np.uint8) if buf else np.zeros(1, np.uint8)
        self._c(lib().locpir_b200_pool_load_queries(
            self.h, raw.ctypes.data, offs.ctypes.data_as(C.POINTER(C.c_uint64)), len(payloads),
            l, _u32(xf), _u32(yf)))

    def load_zero_sheet(self, payload: bytes, regions: int, bits: int, service_values, first: int):
        """ZEROSHEET payload + service values -> encrypted service bits (preprocess_services,
        circuits.hpp:118-146) at slots first + r*bits + j."""
        vals = np.ascontiguousarray(service_values, np.uint64)
        raw = np.frombuffer(payload, np.uint8) if payload else np.zeros(1, np.uint8)
        self._c(lib().locpir_b200_pool_load_zero_sheet(
            self.h, raw.ctypes.data, len(payload), regions, bits,
            vals.ctypes.data_as(C.POINTER(C.c_uint64)), first))

    def store_responses(self, out_first, m: int) -> list:
        """RESPONSE payloads (protocol.hpp:212-227), one bytes object per query."""
        of = np.ascontiguousarray(out_first, np.uint32)
        S = 4 * (self.params.n + 1)
        out = np.zeros(max(1, len(of) * m * S), np.uint8)
        self._c(lib().locpir_b200_pool_store_responses(self.h, _u32(of), len(of), m,
                                                       out.ctypes.data))
        return [out[q * m * S:(q + 1) * m * S].tobytes() for q in range(len(of))]

    # -- client-side encryption on the device (flagged stream) -----
    def client_encrypt(self, lwe_key, seed: int, mus, first_slot: int, first_index: int = 0):
        """Encrypt torus messages into pool slots with the counter-based stream
        (csrc/cbrng.h); bit b -> mu = 0x20000000 if b else 0xE0000000, zero sheet mu = 0."""
        key = np.ascontiguousarray(lwe_key, np.uint8)
        mus = np.ascontiguousarray(mus, np.uint32).reshape(-1)
        self._c(lib().locpir_b200_client_encrypt(self.h, _u8(key), seed, first_index, _u32(mus),
                                                 mus.size, first_slot))

    def debug_blind_rotate(self, lwe_n: np.ndarray) -> np.ndarray:
        """Blind rotation + extraction of combined n-dim LWEs -> N-dim LWEs (pre-KS)."""
        lwe_n = np.ascontiguousarray(lwe_n, np.uint32).reshape(-1, self.params.n + 1)
        out = np.zeros((lwe_n.shape[0], self.params.N + 1), np.uint32)
        self._c(lib().locpir_b200_debug_blind_rotate(self.h, lwe_n.ctypes.data, lwe_n.shape[0],
                                                     out.ctypes.data))
        return out

    def debug_fft_error(self, lwe_n: np.ndarray) -> float:
        """Max |w - rint(w)| over every inverse-transform output of these blind rotations
        (diagnostic kernel instantiation): the FFT rounding margin, exact iff < 1/2."""
        lwe_n = np.ascontiguousarray(lwe_n, np.uint32).reshape(-1, self.params.n + 1)
        e = C.c_double()
        self._c(lib().locpir_b200_debug_fft_error(self.h, lwe_n.ctypes.data, lwe_n.shape[0],
                                                  C.byref(e)))
        return e.value

    def debug_keyswitch(self, lwe_N: np.ndarray) -> np.ndarray:
        lwe_N = np.ascontiguousarray(lwe_N, np.uint32).reshape(-1, self.params.N + 1)
        out = np.zeros((lwe_N.shape[0], self.params.n + 1), np.uint32)
        self._c(lib().locpir_b200_debug_keyswitch(self.h, lwe_N.ctypes.data, lwe_N.shape[0],
                                                  out.ctypes.data))
        return out

    def timing(self, on: bool):
        self._c(lib().locpir_b200_timing_enable(self.h, int(on)))

    def kernel_stats(self):
        ms = (C.c_double * 3)()
        la = (C.c_uint64 * 3)()
        self._c(lib().locpir_b200_kernel_stats(self.h, ms, la))
        return {"blind_rotate": (ms[0], la[0]), "keyswitch": (ms[1], la[1]),
                "linear": (ms[2], la[2])}

    def fp64_peak_tflops(self) -> float:
        v = C.c_double()
        self._c(lib().locpir_b200_fp64_peak(self.h, C.byref(v)))
        return v.value


class Program:
    def __init__(self, ctx: Context, h):
        self.ctx, self.h = ctx, h

    @property
    def kernels(self) -> int:
        return lib().locpir_b200_program_kernels(self.h)

    def launch(self):
        self.ctx._c(lib().locpir_b200_program_launch(self.ctx.h, self.h))

    def prepare(self):
        """Size the context's scratch for this program now (its first launch then
        allocates nothing)."""
        self.ctx._c(lib().locpir_b200_program_prepare(self.ctx.h, self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().locpir_b200_program_destroy(self.h)
            self.h = None

    def __del__(self):
        try:  # interpreter shutdown may already have torn down the module globals
            self.close()
        except Exception:
            pass


def plan(ops) -> dict:
    """Host-only schedule of a gate program (no GPU)."""
    arr = Context.ops_array(ops)
    lv = C.c_uint32()
    br = C.c_uint64()
    ks = C.c_uint64()
    _check(lib().locpir_b200_plan(arr, len(ops), C.byref(lv), C.byref(br), C.byref(ks)))
    return {"levels": lv.value, "blind_rotations": br.value, "key_switches": ks.value}


def check_query_payload(params: "TfheParams", payload: bytes, l: int):
    """Host-only QUERY framing check; raises InvalidArgument with the reference's
    DecodeError message (codec.hpp:180-193, bytes.hpp:118-130)."""
    err = C.create_string_buffer(256)
    raw = np.frombuffer(payload, np.uint8) if payload else np.zeros(1, np.uint8)
    rc = lib().locpir_b200_check_query_payload(C.byref(params.c), raw.ctypes.data, len(payload),
                                               l, err, 256)
    if rc:
        raise InvalidArgument(err.value.decode())


def _tree_mode(xor_tree) -> int:
    """False/0: reference chain, True/1: tree, 2: box-sharded partial (no XOR with Enc(0))."""
    m = int(xor_tree)
    if m not in (0, 1, 2):
        raise ValueError("xor_tree must be 0, 1 or 2")
    return m


def loc_pir_program(Q, R, l, m, x_slots, y_slots, bnd_slots, svc_slots, out_slots,
                    scratch_first, xor_tree=True, maj=False):
    """Host-only emission of the loc_pir gate program (maj=True: flagged majority-borrow
    comparators, locpir_b200_loc_pir_maj_program)."""
    arrs = [np.ascontiguousarray(v, np.uint32).reshape(-1)
            for v in (x_slots, y_slots, bnd_slots, svc_slots, out_slots)]
    cnt = C.c_uint64(0)
    fn = lib().locpir_b200_loc_pir_maj_program if maj else lib().locpir_b200_loc_pir_program
    _check(fn(Q, R, l, m, *[_u32(v) for v in arrs], scratch_first, _tree_mode(xor_tree), None,
              C.byref(cnt)))
    ops = (GateOp * cnt.value)()
    _check(fn(Q, R, l, m, *[_u32(v) for v in arrs], scratch_first, _tree_mode(xor_tree), ops,
              C.byref(cnt)))
    return ops


COMPARATORS = {"reference": 0, "maj": 1, "tree": 2}


def loc_pir_program_ex(Q, R, l, m, x_slots, y_slots, svc_slots, out_slots, scratch_first,
                       bnd_slots=None, boxes_signed=None, xor_tree=True, comparator="reference"):
    """locpir_b200_loc_pir_program_ex: boundaries as pool slots (bnd_slots) or plaintext
    (boxes_signed, folded); comparator "reference" | "maj" | "tree" (flagged modes)."""
    if (bnd_slots is None) == (boxes_signed is None):
        raise ValueError("give exactly one of bnd_slots / boxes_signed")
    arrs = [np.ascontiguousarray(v, np.uint32).reshape(-1)
            for v in (x_slots, y_slots, svc_slots, out_slots)]
    bnd = None if bnd_slots is None else np.ascontiguousarray(bnd_slots, np.uint32).reshape(-1)
    bx = None if boxes_signed is None else np.ascontiguousarray(boxes_signed, np.int64).reshape(-1)
    args = (Q, R, l, m, _u32(arrs[0]), _u32(arrs[1]), _u32(bnd) if bnd is not None else None,
            bx.ctypes.data_as(C.POINTER(C.c_int64)) if bx is not None else None,
            _u32(arrs[2]), _u32(arrs[3]), scratch_first, _tree_mode(xor_tree),
            COMPARATORS[comparator])
    cnt = C.c_uint64(0)
    _check(lib().locpir_b200_loc_pir_program_ex(*args, None, C.byref(cnt)))
    ops = (GateOp * cnt.value)()
    _check(lib().locpir_b200_loc_pir_program_ex(*args, ops, C.byref(cnt)))
    return ops


def loc_pir_folded_program(Q, R, l, m, x_slots, y_slots, boxes_signed, svc_slots, out_slots,
                           scratch_first, xor_tree=True):
    """Flagged mode: loc_pir against PLAINTEXT box boundaries
    (dataset.hpp:250-253 makes them trivial words), comparators constant-folded.
    boxes_signed: [R, 4] (x1, x2, y1, y2) signed l-bit grid values."""
    arrs = [np.ascontiguousarray(v, np.uint32).reshape(-1)
            for v in (x_slots, y_slots, svc_slots, out_slots)]
    bx = np.ascontiguousarray(boxes_signed, np.int64).reshape(-1)
    if bx.size != 4 * R:
        raise ValueError("boxes_signed must hold R x 4 values")
    bxp = bx.ctypes.data_as(C.POINTER(C.c_int64))
    cnt = C.c_uint64(0)
    args = (Q, R, l, m, _u32(arrs[0]), _u32(arrs[1]), bxp, _u32(arrs[2]), _u32(arrs[3]),
            scratch_first, _tree_mode(xor_tree))
    _check(lib().locpir_b200_loc_pir_folded_program(*args, None, C.byref(cnt)))
    ops = (GateOp * cnt.value)()
    _check(lib().locpir_b200_loc_pir_folded_program(*args, ops, C.byref(cnt)))
    return ops


# ---------------------------------------------------------------------------
# GateEngine mirror (gate_engine.hpp:130-336)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class CipherBit:
    """One encrypted bit living in a device pool slot (gate_engine.hpp:81-109)."""
    engine_id: int
    slot: int
    epoch: int = 0  # slot-arena generation (GateEngine.reset_slots)

    def kind(self) -> str:
        return "tfhe-b200"


class GateEngine:
    _ids = itertools.count(1)

    def __init__(self, ctx: Context, keys: ClientKeys, seed: int):
        self.ctx = ctx
        self.keys = keys
        self.params = keys.params
        self._id = next(GateEngine._ids)
        self._seed = seed
        self._enc_counter = 0
        self._next_slot = 0
        self._epoch = 0
        self._limit = 0xFFFFFFF0  # first slot this engine may not use
        self._pending: list | None = None
        self._fork_blocks = [0]

    @staticmethod
    def make_b200(keys: ClientKeys, seed: int = 0, device: int = 0, pool: int = 4096):
        ctx = Context(keys.params, device)
        ctx.upload_keys(keys.bk, keys.ksk)
        ctx.pool_reserve(pool)
        return GateEngine(ctx, keys, seed)

    # -- bookkeeping -----------------------------------------------------------
    def kind(self) -> str:
        return "tfhe-b200"

    def fork(self, lane: int) -> "GateEngine":
        # deterministic bootstrap: nothing to fork.  The mirror is not
        # thread-safe (one host thread per engine, like a reference GateEngine,
        # gate_engine.hpp:335); the C++ integration header supports concurrent forks.
        return self

    def acquire_fork_block(self) -> int:
        b = self._fork_blocks[0]
        self._fork_blocks[0] += 1
        return b

    def secret_key(self):
        return self.keys.lwe_key

    def counters(self) -> dict:
        self.flush()
        return self.ctx.counters()

    def counters_reset(self):
        self.ctx.counters_reset()

    def reset_slots(self):
        """Slot arena: every gate output owns one pool slot until this call; a long-running
        caller resets between independent evaluations.  Older bits are then rejected."""
        self.flush()
        self._next_slot = 0
        self._epoch += 1

    def slots_in_use(self) -> int:
        return self._next_slot

    def reserve_server_tail(self, headroom: int = 1 << 16) -> int:
        """Cap this engine below the returned slot and hand the pool tail to a
        BatchingServer on the same context (BatchingServer(..., base_slot=...))."""
        self.flush()
        self._limit = min(self._limit, self._next_slot + headroom)
        return self._limit

    def _alloc(self, k: int = 1) -> int:
        s = self._next_slot
        if s + k > self._limit:
            raise LogicError(f"engine slot range exhausted at slot {s} (reset_slots() between "
                             "evaluations, or a server owns the pool tail)")
        self._next_slot += k
        if self._next_slot > self.ctx.pool_capacity:
            self.flush()
            self.ctx.pool_reserve(min(self._limit, max(self._next_slot, 2 * self.ctx.pool_capacity)))
        return s

    def _bit(self, c: CipherBit) -> int:
        if not isinstance(c, CipherBit) or c.engine_id != self._id:
            raise InvalidArgument("cipher bit belongs to a different engine")
        if c.epoch != self._epoch:
            raise InvalidArgument("cipher bit predates reset_slots()")
        return c.slot

    def _emit(self, kind, a=_abi.SLOT_NONE, b=_abi.SLOT_NONE, c=_abi.SLOT_NONE) -> CipherBit:
        out = self._alloc()
        op = (kind, a, b, c, out)
        if self._pending is not None:
            self._pending.append(op)
        else:
            self.ctx.run([op])
        return CipherBit(self._id, out, self._epoch)

    @contextlib.contextmanager
    def batch(self):
        """Record gates and run them level-batched on exit (the circuit scheduler)."""
        outer = self._pending is not None
        if not outer:
            self._pending = []
        try:
            yield self
        finally:
            if not outer:
                self.flush()

    def flush(self):
        if self._pending:
            ops, self._pending = self._pending, []
            self.ctx.run(ops)
        elif self._pending is not None:
            pass

    # -- client-side helpers ----------------------------------------------------
    def constant(self, b: bool) -> CipherBit:
        return self._emit(_abi.CONST, 1 if b else 0)

    def encrypt(self, b: bool) -> CipherBit:
        return self.encrypt_many([b])[0]

    def encrypt_many(self, bits) -> list:
        bits = list(bits)
        cts = self.keys.encrypt_bits(bits, self._seed + self._enc_counter)
        self._enc_counter += 1
        return self.load(cts)

    def load(self, cts: np.ndarray) -> list:
        cts = np.asarray(cts, np.uint32).reshape(-1, self.params.n + 1)
        self.flush()
        first = self._alloc(cts.shape[0])
        self.ctx.h2d(first, cts)
        return [CipherBit(self._id, first + i, self._epoch) for i in range(cts.shape[0])]

    def sample(self, c: CipherBit) -> np.ndarray:
        self.flush()
        return self.ctx.d2h(self._bit(c), 1)[0]

    def samples(self, bits) -> np.ndarray:
        self.flush()
        slots = [self._bit(c) for c in bits]
        if not slots:
            return np.zeros((0, self.params.n + 1), np.uint32)
        lo, hi = min(slots), max(slots)
        block = self.ctx.d2h(lo, hi - lo + 1)
        return block[[s - lo for s in slots]]

    def decrypt(self, c: CipherBit) -> bool:
        return bool(self.keys.decrypt_bits(self.sample(c))[0])

    def decrypt_many(self, bits) -> np.ndarray:
        return self.keys.decrypt_bits(self.samples(bits))

    # -- gates (gate_engine.hpp:196-269) -----------------------------------------
    def hom_and(self, a, b):
        return self._emit(_abi.AND, self._bit(a), self._bit(b))

    def hom_or(self, a, b):
        return self._emit(_abi.OR, self._bit(a), self._bit(b))

    def hom_xor(self, a, b):
        return self._emit(_abi.XOR, self._bit(a), self._bit(b))

    def hom_xnor(self, a, b):
        return self._emit(_abi.XNOR, self._bit(a), self._bit(b))

    def hom_nand(self, a, b):
        return self._emit(_abi.NAND, self._bit(a), self._bit(b))

    def hom_nor(self, a, b):
        return self._emit(_abi.NOR, self._bit(a), self._bit(b))

    def hom_not(self, a):
        return self._emit(_abi.NOT, self._bit(a))

    def hom_mux(self, sel, a, b):
        return self._emit(_abi.MUX, self._bit(sel), self._bit(a), self._bit(b))

    def hom_maj(self, a, b, c):
        """3-input majority in one bootstrap (flagged; not in the reference gate set)."""
        return self._emit(_abi.MAJ, self._bit(a), self._bit(b), self._bit(c))

    def hom_xor3(self, a, b, c):
        """a ^ b ^ c in one bootstrap (flagged; not in the reference gate set)."""
        return self._emit(_abi.XOR3, self._bit(a), self._bit(b), self._bit(c))
