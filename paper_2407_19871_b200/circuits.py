"""Python mirror of the reference codec and circuits over the B200 engine.

Follows codec.hpp:16-157 (fixed-point words, LSB at index 0) and
circuits.hpp:187-324 (comparator, masking, XOR-sum, loc_pir) gate for gate, so
gate counts match N(12l + 2m + 3) (bench.hpp:35-43).  Gates are recorded inside
``engine.batch()`` and run level-batched by the C++ circuit scheduler.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .engine import CipherBit, GateEngine, InvalidArgument


@dataclass(frozen=True)
class FixedPointFormat:
    """codec.hpp:16-34 (default 9 + 7 bits)."""
    int_bits: int = 9
    frac_bits: int = 7

    def total_bits(self) -> int:
        return self.int_bits + self.frac_bits

    def validate(self):
        if self.int_bits < 1:
            raise InvalidArgument("fixed-point format needs a sign bit")
        if self.total_bits() < 2 or self.total_bits() > 63:
            raise InvalidArgument("fixed-point width out of range")


def format_for_length(l: int) -> FixedPointFormat:
    """bench.hpp:331-335."""
    ib = min(9, l - 1)
    return FixedPointFormat(ib, l - ib)


@dataclass
class PlainWord:
    """codec.hpp:50-86: two's complement bits, index 0 = LSB."""
    bits: list
    format: FixedPointFormat

    def signed_value(self) -> int:
        l = len(self.bits)
        u = sum(1 << i for i, b in enumerate(self.bits) if b)
        return u - (1 << l) if self.bits[l - 1] else u

    @staticmethod
    def from_integer(v: int, fmt: FixedPointFormat) -> "PlainWord":
        fmt.validate()
        l = fmt.total_bits()
        if v < -(1 << (l - 1)) or v > (1 << (l - 1)) - 1:
            raise IndexError(f"value does not fit in {l} bits")
        u = v & ((1 << l) - 1)
        return PlainWord([(u >> i) & 1 for i in range(l)], fmt)

    @staticmethod
    def from_pattern(pattern: int, l: int, fmt: FixedPointFormat) -> "PlainWord":
        return PlainWord([(pattern >> i) & 1 for i in range(l)], fmt)


@dataclass
class CipherWord:
    """codec.hpp:106-109."""
    bits: list
    format: FixedPointFormat


@dataclass
class ServiceCiphertext:
    bits: list = field(default_factory=list)


@dataclass
class EncodedRegion:
    """circuits.hpp:22-27: half-open [x1, x2) x [y1, y2) plus the service."""
    x1: CipherWord
    x2: CipherWord
    y1: CipherWord
    y2: CipherWord
    service: ServiceCiphertext
    region_id: int = 0


def encrypt_word(w: PlainWord, engine: GateEngine) -> CipherWord:
    return CipherWord(engine.encrypt_many(w.bits), w.format)


def constant_word(w: PlainWord, engine: GateEngine) -> CipherWord:
    with engine.batch():
        bits = [engine.constant(bool(b)) for b in w.bits]
    return CipherWord(bits, w.format)


def decrypt_word(cw: CipherWord, engine: GateEngine) -> PlainWord:
    return PlainWord([int(b) for b in engine.decrypt_many(cw.bits)], cw.format)


def trivial_services(values, m: int, engine: GateEngine):
    out = []
    with engine.batch():
        for v in values:
            if m < 64 and v >> m:
                raise IndexError("service value does not fit")
            out.append(ServiceCiphertext([engine.constant(bool((v >> j) & 1)) for j in range(m)]))
    return out


def decrypt_service(s: ServiceCiphertext, engine: GateEngine) -> int:
    bits = engine.decrypt_many(s.bits)
    return sum(int(b) << j for j, b in enumerate(bits))


def hom_less(a: CipherWord, b: CipherWord, engine: GateEngine) -> CipherBit:
    """circuits.hpp:191-209."""
    if len(a.bits) != len(b.bits) or a.format != b.format:
        raise InvalidArgument("comparator operands must share length and format")
    if not a.bits:
        raise InvalidArgument("comparator operands must be non-empty")
    l = len(a.bits)
    with engine.batch():
        a_sign = engine.hom_not(a.bits[l - 1])
        b_sign = engine.hom_not(b.bits[l - 1])
        t0 = engine.constant(False)
        for i in range(l):
            ai = a_sign if i + 1 == l else a.bits[i]
            bi = b_sign if i + 1 == l else b.bits[i]
            t1 = engine.hom_xnor(ai, bi)
            t0 = engine.hom_mux(t1, t0, bi)
    return t0


def hom_less_equal(a: CipherWord, b: CipherWord, engine: GateEngine) -> CipherBit:
    """circuits.hpp:212-216."""
    with engine.batch():
        return engine.hom_not(hom_less(b, a, engine))


def mask_service(flag: CipherBit, s: ServiceCiphertext, engine: GateEngine) -> ServiceCiphertext:
    """circuits.hpp:219-227."""
    with engine.batch():
        return ServiceCiphertext([engine.hom_and(flag, b) for b in s.bits])


def xor_sum_services(inputs, engine: GateEngine, tree: bool = False) -> ServiceCiphertext:
    """circuits.hpp:240-269: N*m XOR units (chain, or tree + one XOR with Enc(0))."""
    if not inputs:
        return ServiceCiphertext()
    m = len(inputs[0].bits)
    if any(len(s.bits) != m for s in inputs):
        raise InvalidArgument("service ciphertexts must share bit-length")
    out = []
    with engine.batch():
        for j in range(m):
            acc = engine.constant(False)
            if not tree:
                for s in inputs:
                    acc = engine.hom_xor(acc, s.bits[j])
            else:
                lvl = [s.bits[j] for s in inputs]
                while len(lvl) > 1:
                    nxt = [engine.hom_xor(lvl[i], lvl[i + 1]) for i in range(0, len(lvl) - 1, 2)]
                    if len(lvl) & 1:
                        nxt.append(lvl[-1])
                    lvl = nxt
                acc = engine.hom_xor(acc, lvl[0])
            out.append(acc)
    return ServiceCiphertext(out)


def loc_pir(x: CipherWord, y: CipherWord, regions, engine: GateEngine,
            workers: int = 1, tree: bool = False) -> ServiceCiphertext:
    """circuits.hpp:276-324; `workers` is accepted for API parity (the GPU batches)."""
    if not regions:
        return ServiceCiphertext()
    if x.format != y.format:
        raise InvalidArgument("coordinate words must share a format")
    m = len(regions[0].service.bits)
    for r in regions:
        if not (r.x1.format == x.format and r.x2.format == x.format and
                r.y1.format == y.format and r.y2.format == y.format):
            raise InvalidArgument("region boundary format mismatch")
        if len(r.service.bits) != m:
            raise InvalidArgument("regions must share the service bit-length")
    with engine.batch():
        masked = []
        for r in regions:
            x_l = hom_less_equal(r.x1, x, engine)
            x_r = hom_less(x, r.x2, engine)
            y_l = hom_less_equal(r.y1, y, engine)
            y_r = hom_less(y, r.y2, engine)
            v1 = engine.hom_and(x_l, x_r)
            v2 = engine.hom_and(y_l, y_r)
            f = engine.hom_and(v1, v2)
            masked.append(mask_service(f, r.service, engine))
        return xor_sum_services(masked, engine, tree)


def predict_gate_units(regions: int, word_bits: int, service_bits: int) -> int:
    """bench.hpp:35-43."""
    if regions == 0 or word_bits == 0 or service_bits == 0:
        raise InvalidArgument("gate prediction needs positive arguments")
    return regions * (12 * word_bits + 2 * service_bits + 3)
