"""ctypes view of the CPU oracle (oracle/tfhe_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2407_19871_b200) never imports this module.

Reference anchors (see tfhe_oracle.h for the full list): torus.hpp:19-222 (LWE
layer), gate_engine.hpp:117-269 (gates), circuits.hpp:187-324 (circuits).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")

EXACT, FFT = 0, 1
GATES = {"and": 0, "or": 1, "xor": 2, "xnor": 3, "nand": 4, "mux": 5, "not": 6, "nor": 7,
         "andny": 10, "orny": 11, "maj": 12, "xor3": 13}


class GateItem(C.Structure):
    _fields_ = [("kind", C.c_int), ("a", C.c_void_p), ("b", C.c_void_p), ("c", C.c_void_p),
                ("out", C.c_void_p)]


class Params(C.Structure):
    _fields_ = [("n", C.c_uint32), ("N", C.c_uint32), ("k", C.c_uint32), ("l", C.c_uint32),
                ("bgbit", C.c_uint32), ("t", C.c_uint32), ("basebit", C.c_uint32),
                ("alpha_in", C.c_double), ("alpha_bk", C.c_double)]


class KeySet(C.Structure):
    _fields_ = [("p", Params), ("lwe_key", C.POINTER(C.c_uint8)),
                ("trlwe_key", C.POINTER(C.c_uint8)), ("bk", C.POINTER(C.c_uint32)),
                ("ksk", C.POINTER(C.c_uint32)), ("bk_fft", C.POINTER(C.c_double)),
                ("bk_fft_soa", C.POINTER(C.c_double))]


class Sampler(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int), ("sigma", C.c_double)]


def build():
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.environ.get("LOCPIR_ORACLE_LIB", LIB_PATH)  # bench.py: the AVX-512 build
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        u32p = C.POINTER(C.c_uint32)
        u8p = C.POINTER(C.c_uint8)
        L.or_keyset_generate.argtypes = [C.POINTER(KeySet), C.POINTER(Params), C.c_uint64]
        L.or_keyset_free.argtypes = [C.POINTER(KeySet)]
        L.or_params_default.argtypes = [C.c_int, C.POINTER(Params)]
        L.or_bk_words.argtypes = [C.POINTER(Params)]
        L.or_bk_words.restype = C.c_size_t
        L.or_ksk_words.argtypes = [C.POINTER(Params)]
        L.or_ksk_words.restype = C.c_size_t
        L.or_keygen.argtypes = [C.c_uint32, C.c_uint64, u8p]
        L.or_sampler_init.argtypes = [C.POINTER(Sampler), C.c_uint64, C.c_double]
        L.or_sampler_uniform.argtypes = [C.POINTER(Sampler)]
        L.or_sampler_uniform.restype = C.c_uint32
        L.or_sampler_gaussian.argtypes = [C.POINTER(Sampler)]
        L.or_sampler_gaussian.restype = C.c_uint32
        L.or_encrypt_torus.argtypes = [C.c_uint32, u8p, C.c_uint32, C.POINTER(Sampler), u32p]
        L.or_encrypt_bit.argtypes = [C.c_int, u8p, C.c_uint32, C.POINTER(Sampler), u32p]
        L.or_phase.argtypes = [u32p, u8p, C.c_uint32]
        L.or_phase.restype = C.c_uint32
        L.or_decrypt_bit.argtypes = [u32p, u8p, C.c_uint32]
        L.or_bootstrap_standin.argtypes = [u32p, u8p, C.c_uint32, C.POINTER(Sampler), u32p]
        L.or_fft_tables.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_fft_forward_i32.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p]
        L.or_fft_inverse_add.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p]
        L.or_fft_margin.argtypes = [C.c_int]
        L.or_fft_margin.restype = C.c_double
        L.or_polymul_exact_add.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_decompose.argtypes = [C.POINTER(Params), u32p, C.c_uint32, C.c_void_p]
        L.or_mod_switch.argtypes = [C.c_uint32, C.c_uint32]
        L.or_mod_switch.restype = C.c_uint32
        L.or_blind_rotate_extract.argtypes = [C.POINTER(KeySet), u32p, C.c_uint32, C.c_int, u32p]
        L.or_blind_rotate_acc.argtypes = [C.POINTER(KeySet), u32p, C.c_uint32, C.c_int,
                                          C.c_uint32, u32p]
        L.or_external_product.argtypes = [C.POINTER(KeySet), C.c_uint32, u32p, C.c_int, u32p]
        L.or_keyswitch.argtypes = [C.POINTER(KeySet), u32p, u32p]
        L.or_gate.argtypes = [C.POINTER(KeySet), C.c_int, u32p, u32p, u32p, C.c_int, u32p]
        L.or_cb_encrypt.argtypes = [u8p, C.c_uint32, C.c_uint64, C.c_uint32, u32p, C.c_uint64,
                                    C.c_double, u32p]
        L.or_cb_encrypt.restype = None
        L.or_cb_philox.argtypes = [u32p, C.c_uint64, u32p]
        L.or_cb_philox.restype = None
        L.or_cb_log.argtypes = [C.c_double]
        L.or_cb_log.restype = C.c_double
        L.or_cb_cos2pi.argtypes = [C.c_double]
        L.or_cb_cos2pi.restype = C.c_double
        L.or_cb_noise.argtypes = [C.c_uint64, C.c_uint32, C.c_double]
        L.or_cb_noise.restype = C.c_uint32
        L.or_gate_list.argtypes = [C.POINTER(KeySet), C.POINTER(GateItem), C.c_uint64, C.c_int,
                                   C.c_int]
        L.or_gate_batch.argtypes = [C.POINTER(KeySet), C.c_int, u32p, u32p, u32p, C.c_uint64,
                                    C.c_int, C.c_int]
        L.or_gate_batch_simd.argtypes = [C.POINTER(KeySet), C.c_int, u32p, u32p, u32p,
                                         C.c_uint64, C.c_int]
        L.or_simd_lanes.restype = C.c_int
        L.or_gate_list_simd.argtypes = [C.POINTER(KeySet), C.POINTER(GateItem), C.c_uint64,
                                        C.c_int]
        _lib = L
    return _lib


def simd_lanes() -> int:
    """Ciphertexts per SIMD lane group of gate_batch_simd (8 with AVX-512, 4 with AVX2)."""
    return int(lib().or_simd_lanes())


def _u32(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def params(level: int) -> Params:
    p = Params()
    lib().or_params_default(level, C.byref(p))
    return p


def keygen_bits(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n, np.uint8)
    lib().or_keygen(n, seed, _u8(out))
    return out


class NoiseSampler:
    """torus.hpp:119-138 restated in C."""

    def __init__(self, seed: int, sigma: float):
        self.s = Sampler()
        lib().or_sampler_init(C.byref(self.s), seed, sigma)

    def uniform(self) -> int:
        return lib().or_sampler_uniform(C.byref(self.s))

    def gaussian(self) -> int:
        return lib().or_sampler_gaussian(C.byref(self.s))


def encrypt_bit(bit: int, key: np.ndarray, sampler: NoiseSampler) -> np.ndarray:
    out = np.zeros(len(key) + 1, np.uint32)
    lib().or_encrypt_bit(int(bit), _u8(key), len(key), C.byref(sampler.s), _u32(out))
    return out


def encrypt_torus(mu: int, key: np.ndarray, sampler: NoiseSampler) -> np.ndarray:
    out = np.zeros(len(key) + 1, np.uint32)
    lib().or_encrypt_torus(mu, _u8(key), len(key), C.byref(sampler.s), _u32(out))
    return out


def phase(ct: np.ndarray, key: np.ndarray) -> int:
    ct = np.ascontiguousarray(ct, np.uint32)
    return lib().or_phase(_u32(ct), _u8(key), len(key))


def decrypt_bit(ct: np.ndarray, key: np.ndarray) -> int:
    ct = np.ascontiguousarray(ct, np.uint32)
    return int(lib().or_decrypt_bit(_u32(ct), _u8(key), len(key)))


def bootstrap_standin(ct, key, sampler) -> np.ndarray:
    ct = np.ascontiguousarray(ct, np.uint32)
    out = np.zeros(len(key) + 1, np.uint32)
    lib().or_bootstrap_standin(_u32(ct), _u8(key), len(key), C.byref(sampler.s), _u32(out))
    return out


def fft_tables(N: int):
    W = np.zeros((N // 4, 2))
    TW = np.zeros((N // 2, 2))
    UT = np.zeros((N // 2, 2))
    lib().or_fft_tables(N, W.ctypes.data, TW.ctypes.data, UT.ctypes.data)
    return W, TW, UT


def fft_forward(d: np.ndarray) -> np.ndarray:
    d = np.ascontiguousarray(d, np.int32)
    out = np.zeros((len(d) // 2, 2))
    lib().or_fft_forward_i32(len(d), d.ctypes.data, out.ctypes.data)
    return out


def fft_inverse_add(F: np.ndarray, acc: np.ndarray) -> None:
    F = np.array(F, np.float64, copy=True)
    lib().or_fft_inverse_add(len(acc), F.ctypes.data, acc.ctypes.data)


def fft_margin(reset: bool = True) -> float:
    """Max distance from an integer of any inverse-transform output before rounding since
    the last reset (the FFT rounding margin; exact while < 1/2)."""
    return lib().or_fft_margin(1 if reset else 0)


def polymul_exact_add(d: np.ndarray, b: np.ndarray, acc: np.ndarray) -> None:
    d = np.ascontiguousarray(d, np.int32)
    b = np.ascontiguousarray(b, np.uint32)
    lib().or_polymul_exact_add(len(acc), d.ctypes.data, b.ctypes.data, acc.ctypes.data)


def mod_switch(x: int, N: int) -> int:
    return lib().or_mod_switch(x, N)


class TfheKeys:
    """Seeded TFHE key set (LWE key, TRLWE key, BK, KSK) -- oracle derivation."""

    def __init__(self, level: int = 128, seed: int = 1, p: Params | None = None):
        self.ks = KeySet()
        self.p = p if p is not None else params(level)
        rc = lib().or_keyset_generate(C.byref(self.ks), C.byref(self.p), seed)
        if rc:
            raise RuntimeError(f"or_keyset_generate failed: {rc}")
        n, N = self.p.n, self.p.N
        self.n, self.N = n, N
        self.lwe_key = np.ctypeslib.as_array(self.ks.lwe_key, (n,)).copy()
        self.trlwe_key = np.ctypeslib.as_array(self.ks.trlwe_key, (N,)).copy()
        self.bk_words = lib().or_bk_words(C.byref(self.p))
        self.ksk_words = lib().or_ksk_words(C.byref(self.p))

    def bk(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.ks.bk, (self.bk_words,))

    def ksk(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.ks.ksk, (self.ksk_words,))

    def bk_fft(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.ks.bk_fft, (self.bk_words,))

    def __del__(self):
        try:
            lib().or_keyset_free(C.byref(self.ks))
        except Exception:
            pass

    # -- client side -------------------------------------------------------
    def encrypt(self, bit: int, sampler: NoiseSampler) -> np.ndarray:
        return encrypt_bit(bit, self.lwe_key, sampler)

    def decrypt(self, ct: np.ndarray) -> int:
        return decrypt_bit(ct, self.lwe_key)

    def phase(self, ct: np.ndarray) -> int:
        return phase(ct, self.lwe_key)

    # -- server side (oracle evaluation) -----------------------------------
    def gate(self, kind: str, a, b=None, c=None, mode: int = FFT) -> np.ndarray:
        out = np.zeros(self.n + 1, np.uint32)
        a = np.ascontiguousarray(a, np.uint32)
        bb = np.ascontiguousarray(b, np.uint32) if b is not None else None
        cc = np.ascontiguousarray(c, np.uint32) if c is not None else None
        rc = lib().or_gate(C.byref(self.ks), GATES[kind], _u32(a),
                           _u32(bb) if bb is not None else None,
                           _u32(cc) if cc is not None else None, mode, _u32(out))
        if rc:
            raise ValueError(f"oracle gate {kind} failed: {rc}")
        return out

    def gate_batch(self, kind: str, a: np.ndarray, b: np.ndarray, mode: int = FFT,
                   threads: int = 1) -> np.ndarray:
        a = np.ascontiguousarray(a, np.uint32)
        b = np.ascontiguousarray(b, np.uint32)
        out = np.zeros_like(a)
        rc = lib().or_gate_batch(C.byref(self.ks), GATES[kind], _u32(a), _u32(b), _u32(out),
                                 a.shape[0], mode, threads)
        if rc:
            raise ValueError(f"oracle gate batch failed: {rc}")
        return out

    def gate_batch_simd(self, kind: str, a: np.ndarray, b: np.ndarray,
                        threads: int = 1) -> np.ndarray:
        """FFT-mode 2-input gates, 4 ciphertexts per AVX2 lane group: bit-identical to
        gate_batch(kind, a, b, FFT) (the CPU baseline's fast path)."""
        a = np.ascontiguousarray(a, np.uint32)
        b = np.ascontiguousarray(b, np.uint32)
        out = np.zeros_like(a)
        rc = lib().or_gate_batch_simd(C.byref(self.ks), GATES[kind], _u32(a), _u32(b),
                                      _u32(out), a.shape[0], threads)
        if rc:
            raise ValueError(f"oracle simd gate batch failed: {rc}")
        return out

    def blind_rotate_extract(self, lwe: np.ndarray, mu: int = 0x20000000,
                             mode: int = FFT) -> np.ndarray:
        lwe = np.ascontiguousarray(lwe, np.uint32)
        out = np.zeros(self.N + 1, np.uint32)
        lib().or_blind_rotate_extract(C.byref(self.ks), _u32(lwe), mu, mode, _u32(out))
        return out

    def blind_rotate_acc(self, lwe, mu=0x20000000, mode=FFT, steps=0xFFFFFFFF) -> np.ndarray:
        lwe = np.ascontiguousarray(lwe, np.uint32)
        out = np.zeros(2 * self.N, np.uint32)
        lib().or_blind_rotate_acc(C.byref(self.ks), _u32(lwe), mu, mode, steps, _u32(out))
        return out

    def external_product(self, i: int, trlwe: np.ndarray, mode: int = FFT) -> np.ndarray:
        trlwe = np.ascontiguousarray(trlwe, np.uint32)
        out = np.zeros(2 * self.N, np.uint32)
        lib().or_external_product(C.byref(self.ks), i, _u32(trlwe), mode, _u32(out))
        return out

    def keyswitch(self, lweN: np.ndarray) -> np.ndarray:
        lweN = np.ascontiguousarray(lweN, np.uint32)
        out = np.zeros(self.n + 1, np.uint32)
        lib().or_keyswitch(C.byref(self.ks), _u32(lweN), _u32(out))
        return out

    def decompose(self, x: np.ndarray, level: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.uint32)
        out = np.zeros(self.N, np.int32)
        lib().or_decompose(C.byref(self.p), _u32(x), level, out.ctypes.data)
        return out


# gate-program kinds (include/locpir_b200.h) -> oracle kinds; NOT/COPY/CONST are free
_PROG_BOOT = {0: 0, 1: 1, 2: 2, 3: 3, 4: 4, 5: 5, 7: 7, 10: 10, 11: 11, 12: 12, 13: 13}
_NOT, _COPY, _CONST = 6, 8, 9


def run_program(K: "TfheKeys", ops, pool: np.ndarray, threads: int = 1, mode: int = FFT,
                simd=False):
    """Evaluates a gate program (5-tuples or ctypes GateOps over pool slots, the layout of
    include/locpir_b200.h) on the oracle: bootstrapped gates level by level, each level
    one threaded or_gate_list call (simd=True: or_gate_list_simd, FFT mode, blind
    rotations lane-batched, bit-identical; simd="auto": per level, whichever of the two
    is faster for its width); free gates in program order between levels.
    pool: [slots, n+1] uint32, updated in place.  Test / baseline infrastructure."""
    SLOT_NONE = 0xFFFFFFFF
    ops = [(o.kind, o.in0, o.in1, o.in2, o.out) if not isinstance(o, tuple) else o for o in ops]
    lvl = {}
    levels = {}
    for i, (k, a, b, c, o) in enumerate(ops):
        ins = [s for s in (a, b, c) if s != SLOT_NONE] if k != _CONST else []
        base = max((lvl.get(s, 0) for s in ins), default=0)
        L = base + 1 if k in _PROG_BOOT else base
        lvl[o] = L
        levels.setdefault(L, []).append(i)
    row = pool.strides[0]
    base_ptr = pool.ctypes.data
    n = pool.shape[1] - 1
    for L in sorted(levels):
        idx = levels[L]
        boot = [i for i in idx if ops[i][0] in _PROG_BOOT]
        if boot:
            items = (GateItem * len(boot))()
            for j, i in enumerate(boot):
                k, a, b, c, o = ops[i]
                items[j] = GateItem(_PROG_BOOT[k], base_ptr + a * row,
                                    base_ptr + b * row if b != SLOT_NONE else None,
                                    base_ptr + c * row if c != SLOT_NONE else None,
                                    base_ptr + o * row)
            # lane-batching pays once the level fills the lanes of the threads: a lane
            # group of L rotations costs ~L/3 scalar gates with AVX-512 (measured ~3x per
            # gate), so narrow levels (single queries) stay on the scalar path
            nb = len(boot)
            L = simd_lanes()
            t_scalar = -(-nb // threads)
            t_simd = -(-nb // (threads * L)) * L / 3.0
            if mode == FFT and (simd is True or (simd == "auto" and t_simd < t_scalar)):
                rc = lib().or_gate_list_simd(C.byref(K.ks), items, nb,
                                             min(threads, -(-nb // L)))
            else:
                rc = lib().or_gate_list(C.byref(K.ks), items, len(boot), mode, threads)
            if rc:
                raise ValueError(f"oracle gate list failed: {rc}")
        for i in idx:
            k, a, b, c, o = ops[i]
            if k == _NOT:
                pool[o] = (0 - pool[a].astype(np.int64)) & 0xFFFFFFFF
            elif k == _COPY:
                pool[o] = pool[a]
            elif k == _CONST:
                pool[o] = 0
                pool[o, n] = 0x20000000 if a else 0xE0000000
    return pool


def cb_encrypt(key: np.ndarray, seed: int, first_index: int, mus, alpha: float) -> np.ndarray:
    """Counter-based client encryption (cbrng.h stream) of torus messages `mus`."""
    mus = np.ascontiguousarray(mus, np.uint32).reshape(-1)
    key = np.ascontiguousarray(key, np.uint8)
    out = np.zeros((mus.size, key.size + 1), np.uint32)
    lib().or_cb_encrypt(_u8(key), key.size, seed, first_index, _u32(mus), mus.size, alpha, _u32(out))
    return out


def cb_philox(ctr, seed: int) -> list:
    c = np.ascontiguousarray(ctr, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().or_cb_philox(_u32(c), seed, _u32(o))
    return [int(v) for v in o]
