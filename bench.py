#!/usr/bin/env python3
"""Benchmark of the hot path: batched TFHE gate bootstrapping on B200.

Workload (BASELINE.json configs[1], the config the headline metric is quoted on):
65,536 independent bootstrapped NAND gates per GPU on seeded uniform encrypted
bits, 128-bit TFHE parameters.  One "step" = one pass of the hot path over that
batch: gate linear form + blind rotation + sample extraction (kernel K1) and key
switching (kernel K2), inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the CPU implementation of the path on the box's host
cores: the oracle port of TFHE gate bootstrapping (oracle/, FP64-FFT mode, all
host threads) -- the reference's own gate "bootstrap" is a secret-key refresh
stand-in (gate_engine.hpp:117-123) whose rate is reported alongside, labelled.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
T_PROCESS = time.perf_counter()  # the wall-budget guard of the stated-size LocPIR runs counts from here
sys.path.insert(0, ROOT)

GATES_PER_GPU = 65536
SECURITY = 128
# seeds follow the reference tools' convention (LOCPIR_SEED, tools/common.hpp:13-28)
KEY_SEED = int(os.environ.get("LOCPIR_SEED", "20240719"), 0)
F_FFT = 5 * 512 * 9 + 6 * 512  # 26,112 flop per 512-point complex transform


def flop_per_br(n=630, k=1, l=3, N=1024):
    """F_BR = n * [((k+1)l + (k+1)) * F_fft + (k+1)^2 l (N/2) 8]."""
    return n * (((k + 1) * l + (k + 1)) * F_FFT + (k + 1) ** 2 * l * (N // 2) * 8)


TRAFFIC_FILES = ("r02_traffic.json", "r01_traffic.json")  # newest committed capture first


def committed_traffic(kernel="k_blind_rotate<3, 7>"):
    """dram__bytes_read.sum + dram__bytes_write.sum of one full-size launch, from the
    newest committed ncu capture (profiles/r0N_traffic.json); None when absent."""
    for f in TRAFFIC_FILES:
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", f)))
            k = d["kernels"][kernel]
            return k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"]
        except Exception:
            continue
    return None


def locpir_roofline(sec, units_per_query, qps, n_gpus, peak_tflops):
    """BASELINE.json: queries/s as a fraction of the bootstrap roofline, the slower of the
    transform arithmetic at the FP64 peak (units x F_BR) and the key bytes at HBM bandwidth
    (|BK_freq| + |KSK| once per GPU: ~19 us, never the binding term)."""
    f_br = flop_per_br(630, 1, 3, 1024) if sec == 128 else flop_per_br(500, 1, 2, 1024)
    roof_qps = n_gpus * peak_tflops * 1e12 / (units_per_query * f_br)
    return {"bound": "fp64", "queries_per_s_roof": roof_qps, "frac": qps / roof_qps,
            "flop_per_unit": f_br}


def hbm_view(G, params, avg_br_ms):
    """K1 against the measured HBM roof: algorithmic and ncu-measured DRAM bytes per launch
    over the launch time (MEASURED_PEAKS.json hbm_gbs)."""
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = None
    alg = G * (2 * 4 * (params.n + 1) + 4 * (params.N + 1)) + params.bk_words() * 8
    t = committed_traffic() if G == GATES_PER_GPU else None
    secs = avg_br_ms * 1e-3
    return {"algorithmic_GBps": alg / secs / 1e9, "dram_GBps": t / secs / 1e9 if t else None,
            "peak_GBps": peak, "frac": (t or alg) / secs / 1e9 / peak if peak else None}


def l1tex_view():
    """The unit that actually binds K1: L1TEX data-pipe utilisation and the
    per-CMux-step wavefront budget, from the newest committed ncu --set full capture
    (profiles/r0N_ncu_blind_rotate.txt); None when absent."""
    for tag in ("r02", "r01"):
        try:
            txt = open(os.path.join(ROOT, "profiles", f"{tag}_ncu_blind_rotate.txt")).read()
        except OSError:
            continue
        m = {}
        for ln in txt.splitlines():
            parts = ln.split()
            if len(parts) == 2 and parts[0].startswith(("l1tex__", "sm__pipe_fp64", "launch__grid")):
                try:
                    m[parts[0]] = float(parts[1])
                except ValueError:
                    pass
        util = m.get("l1tex__throughput.avg.pct_of_peak_sustained_active")
        wf = m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        grid = m.get("launch__grid_size")
        return {"l1tex_utilisation": util / 100 if util else None,
                "fp64_pipe_utilisation": (m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") or 0) / 100 or None,
                "shared_wavefronts_per_cmux_step": wf / (grid * 630) if wf and grid else None,
                "source": f"profiles/{tag}_ncu_blind_rotate.txt (4,736 ciphertexts, 128-bit)",
                "note": "peak is one wavefront per clock per SM; the transform exchanges, BK "
                        "loads and ACC reads keep L1TEX the busiest unit, so 1 - this "
                        "utilisation bounds what better scheduling alone can recover"}
    return None


def keyswitch_view(G, params, avg_ks_ms, ksk_bytes):
    """K2t (ks_tc.cuh) against the INT8 tensor-core roof.  The key switch of a level of G
    ciphertexts is S = A x B with A the (G x K) one-hot digit matrix and B the
    byte-sliced KSK (K x 4(n+1) byte-columns), K = N t 3 (digit values 1..3; d = 0 adds
    nothing): the MMA issues 2 M_pad K N_pad int8 ops (M padded to 256-row CTAs, N to
    256-column tiles).  Peak = 2 x the measured dense bf16
    rate (MEASURED_PEAKS.json; sm_100's kind::i8 runs at twice kind::f16).  The INT32 view
    restates the same launch as the 3/4 x N t (n+1) u32 subtractions the CUDA-core K2 does."""
    secs = avg_ks_ms * 1e-3
    K = params.N * params.c.ks_t * 3
    m_pad = -(-G // 256) * 256
    n_stride = -(-(params.n + 1) // 4) * 4
    n_tiles = -(-(n_stride * 4) // 256)
    ops = 2.0 * m_pad * K * n_tiles * 256
    l2_bytes = (m_pad // 256) * n_tiles * K * 256  # every CTA streams its tile's K x 256 bytes
    adds = G * params.N * params.c.ks_t * (params.n + 1) * 0.75
    int_peak = 148 * 128 * 1.965e9
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        i8_peak, hbm_peak = 2 * peaks["bf16_tflops"] * 1e12, peaks["hbm_gbs"]
        src = "2 x MEASURED_PEAKS.json bf16_tflops (burst)"
    except Exception:
        i8_peak, hbm_peak, src = 4.5e15, None, "nominal B200 dense int8 (no MEASURED_PEAKS.json)"
    dram = committed_traffic("k_keyswitch_tc") if G == GATES_PER_GPU else None
    return {"kernel": "k_keyswitch_tc (K2t, tcgen05.mma kind::i8, TMEM accumulators)",
            "avg_launch_ms": avg_ks_ms,
            "tensor_view": {"bound": "tensor", "achieved_Tops": ops / secs / 1e12,
                            "peak_Tops": i8_peak / 1e12, "frac": ops / secs / i8_peak,
                            "ops_per_launch": ops, "peak_source": src},
            "int32_equivalent": {"adds_Tops": adds / secs / 1e12,
                                 "cuda_core_peak_Tops": int_peak / 1e12,
                                 "note": "the subtractions K2 would do on INT32 lanes "
                                         "(148 SMs x 128 lanes x 1965 MHz)"},
            "l2_view": {"l2_to_smem_bytes_per_launch": l2_bytes,
                        "GBps": l2_bytes / secs / 1e9},
            "hbm_view": {"ksk_bytes": ksk_bytes, "dram_bytes_per_launch": dram,
                         "dram_GBps": dram / secs / 1e9 if dram else None, "peak_GBps": hbm_peak,
                         "note": "the tiled KSK (63 MB at 128-bit) is bulk-copied with evict_last"}}


def workload_config(n_gpus):
    return {
        "workload": "cfg2: 65,536 independent bootstrapped NAND gates per GPU, 128-bit TFHE "
                    "(BASELINE.json configs[1])",
        "gates_per_gpu": GATES_PER_GPU,
        "params": {"n": 630, "N": 1024, "k": 1, "bk_l": 3, "bk_bgbit": 7, "ks_t": 8,
                   "ks_basebit": 2, "alpha_in": "2^-15", "alpha_bk": "2^-25", "torus": "u32"},
        "l2": "inputs 2 x 65,536 x 2,528 B = 331 MB per GPU > 126 MB L2 (no flush needed); "
              "BK_freq 62 MB + KSK 62 MB stay resident by design",
        "parallelism": f"shard{n_gpus}" if n_gpus > 1 else "single",
        "key_seed": KEY_SEED,
    }


# ---------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
_ORACLE_KEYS = {}


def cpu_oracle_rate(budget_s=12.0, threads=None, seed=KEY_SEED):
    """TFHE gate bootstrapping on the host CPU: the oracle's FP64-FFT arithmetic
    (oracle/tfhe_oracle.c) lane-batched -- one ciphertext per SIMD lane, 8 per AVX-512
    vector (4 with AVX2), the bootstrapping-key rows broadcast -- on all host threads with
    the static block partition of parallel.hpp:15-52.  Bit-identical to the scalar port
    (checked on the sample).  Bounded sample."""
    from oracle import oracle as O
    threads = threads or os.cpu_count() or 1
    K = _ORACLE_KEYS.get((SECURITY, seed))
    if K is None:  # key generation is setup, not part of any timed sample
        K = _ORACLE_KEYS[(SECURITY, seed)] = O.TfheKeys(SECURITY, seed)
    s = O.NoiseSampler(seed + 1, K.p.alpha_in)
    lanes = O.simd_lanes()
    ca = np.stack([K.encrypt(1, s) for _ in range(lanes)])
    cb = np.stack([K.encrypt(1, s) for _ in range(lanes)])
    t = time.perf_counter()
    K.gate_batch("nand", ca[:1], cb[:1], O.FFT, 1)
    t_scalar = time.perf_counter() - t
    t = time.perf_counter()
    K.gate_batch_simd("nand", ca, cb, 1)
    t_group = time.perf_counter() - t
    per_thread = lanes * max(1, int(budget_s / max(t_group, 1e-3)))
    count = threads * per_thread
    rng = np.random.default_rng(seed)
    A = rng.integers(0, 2, count)
    B = rng.integers(0, 2, count)
    a = np.stack([K.encrypt(int(x), s) for x in A])
    b = np.stack([K.encrypt(int(x), s) for x in B])
    t = time.perf_counter()
    out = K.gate_batch_simd("nand", a, b, threads)
    dt = time.perf_counter() - t
    ok = all(K.decrypt(out[i]) == 1 - (A[i] & B[i]) for i in range(0, count, max(1, count // 64)))
    same = bool(np.array_equal(out[:2], K.gate_batch("nand", a[:2], b[:2], O.FFT, 2)))
    return {"value": count / dt, "unit": "gates/s", "cores": threads, "kind": "port",
            "sample": f"{count} NAND gates (128-bit TFHE, FP64-FFT oracle port lane-batched "
                      f"{lanes} ciphertexts per SIMD vector, {threads} threads, {dt:.1f} s, "
                      f"build {ORACLE_BUILD})",
            "gates": count, "seconds": dt,
            "ms_per_gate_per_core": 1e3 * dt * threads / count,
            "scalar_port_ms_per_gate_per_core": 1e3 * t_scalar,
            "tfhe11_ms_per_gate_per_core": 13.0,  # PAPER.md:78 (TFHE 1.1, one core)
            "bit_identical_to_scalar_port": same,
            "correct": bool(ok and same)}


def host_cpu():
    """CPU model and core count of the box the baseline ran on."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def standin_rate(threads=None):
    """The reference's own gate refresh stand-in (compiled read-only into oracle/_ref)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if not os.path.exists(exe):
        return None
    threads = threads or os.cpu_count() or 1
    try:
        r = subprocess.run([exe, "standin", "65536", str(threads)], capture_output=True,
                           text=True, timeout=300)
        d = json.loads(r.stdout)
        return {"value": d["gates_per_s"], "unit": "gates/s", "cores": threads,
                "label": "functional stand-in, no bootstrapping (gate_engine.hpp:117-123): "
                         "hom_not(hom_and) with a secret-key re-encryption per gate"}
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


def standin_locpir_rates(threads=None):
    """The reference's own loc_pir (circuits.hpp:276-324) under its refresh-oracle engine on
    its synthetic case at each LocPIR config's shape (compiled read-only into oracle/_ref)."""
    from paper_2407_19871_b200 import workloads as W
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if not os.path.exists(exe):
        return None
    threads = threads or os.cpu_count() or 1
    out = {"label": "functional stand-in, no bootstrapping (gate_engine.hpp:117-123): every "
                    "gate is a secret-key re-encryption, ~1e3-1e4x cheaper than a bootstrap; "
                    "reference parameter sets sec80/sec128", "cores": threads, "configs": {}}
    for name, (sec, Qfull, R, l, m, enc) in W.CONFIGS.items():
        q = {"cfg1": 200, "cfg3": 2, "cfg4": 50, "cfg5": 8}.get(name, 4)
        try:
            r = subprocess.run([exe, "standin_locpir", str(R), str(l), str(m), str(sec), str(q),
                                str(threads)], capture_output=True, text=True, timeout=300)
            d = json.loads(r.stdout)
            out["configs"][name] = {"queries_per_s": d["queries_per_s"], "queries": q,
                                    "correct": d["wrong"] == 0,
                                    "boundaries": "trivial (the reference encodes regions as "
                                                  "constants)" if enc else "trivial"}
        except Exception as e:  # pragma: no cover
            out["configs"][name] = {"error": str(e)}
    return out


# ---------------------------------------------------------------------------
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    vals = []
    for _ in range(max(0, args.warmup)):
        cpu_oracle_rate(budget_s=2.0, threads=threads)
    for _ in range(args.steps):
        vals.append(cpu_oracle_rate(budget_s=args.ref_budget, threads=threads))
    v = statistics.median([x["value"] for x in vals])
    # one step = one bounded sample of the cfg2 batch (cpu_oracle_rate); ms_per_step is the
    # measured time of the gates actually evaluated in a step, not an extrapolation
    line = {
        "impl": "reference", "metric": "bootstrapped gates/s (128-bit TFHE)", "value": v,
        "unit": "gates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * statistics.median([x["seconds"] for x in vals]),
        "gates_per_step": statistics.median([x["gates"] for x in vals]),
        "step_note": "each step evaluates a bounded sample (gates_per_step) of the 65,536-gate "
                     "cfg2 batch; value = gates / s over those samples",
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.gpus),
        "cpu_baseline": {"value": v, "unit": "gates/s", "cores": threads, "kind": "port",
                         "sample": vals[-1]["sample"] + f"; median of {args.steps} steps",
                         "ms_per_gate_per_core": vals[-1]["ms_per_gate_per_core"],
                         "scalar_port_ms_per_gate_per_core":
                             vals[-1]["scalar_port_ms_per_gate_per_core"],
                         "bit_identical_to_scalar_port":
                             all(x["bit_identical_to_scalar_port"] for x in vals),
                         "tfhe11_ms_per_gate_per_core": 13.0, "host_cpu": host_cpu()},
        "e2e": {"value": v, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "The reference contains no gate bootstrapping (TFHE 1.1 is absent from "
                "/root/reference); the timed CPU path is the oracle port of the TFHE "
                "algorithm, lane-batched over SIMD vectors (bit-identical to the scalar "
                "port). The reference's own refresh stand-in is reported in "
                "reference_standin.",
        "reference_standin": standin_rate(threads),
    }
    print(json.dumps(line), flush=True)
    return 0


# CPU baseline for the LocPIR configs: (queries, boxes) actually evaluated by the oracle port
CPU_LOCPIR_SAMPLES = {"cfg1": (1, None), "cfg3": (1, 8), "cfg4": (1, 8), "cfg5": (1, 4)}


def cpu_locpir_baseline(threads=None, seed=KEY_SEED):
    """The same loc_pir gate programs evaluated by the oracle port (FP64-FFT mode, blind
    rotations lane-batched over SIMD vectors, bit-identical to the scalar port) level by
    level on all host threads (oracle.run_program), decrypted and checked against the
    plaintext answer.  cfg1 runs in full; cfg3/4/5 run on a box subsample and are
    extrapolated linearly in bootstrap units (SURVEY §8(d) "run cfg3/4/5 on a stated
    subsample and extrapolate linearly")."""
    from oracle import oracle as O
    from paper_2407_19871_b200 import workloads as W
    threads = threads or os.cpu_count() or 1
    out = {}
    keys = {}
    for name, (sec, Qfull, Rfull, l, m, enc) in W.CONFIGS.items():
        Qs, Rs = CPU_LOCPIR_SAMPLES[name]
        Rs = Rs or Rfull
        if sec not in keys:
            keys[sec] = O.TfheKeys(sec, seed)
        K = keys[sec]
        b = W.make_batch(Qs, Rs, l, m, seed=seed + 31 + len(out), encrypted_bounds=enc)
        b.x[0] = (b.boxes[0, 0] + b.boxes[0, 1]) // 2
        b.y[0] = (b.boxes[0, 2] + b.boxes[0, 3]) // 2
        lay = W.PoolLayout(b)
        pool = np.zeros((lay.total, K.n + 1), np.uint32)
        smp = O.NoiseSampler(seed + 7, K.p.alpha_in)
        enc_bits = lambda bits: np.stack([O.encrypt_bit(int(v), K.lwe_key, smp) for v in bits])
        qbits = np.concatenate([W._bits_signed(b.x, l).reshape(-1), W._bits_signed(b.y, l).reshape(-1)])
        pool[lay.x.reshape(-1)] = enc_bits(qbits[: Qs * l])
        pool[lay.y.reshape(-1)] = enc_bits(qbits[Qs * l:])
        bbits = W._bits_signed(b.boxes, l).reshape(-1)
        if enc:
            pool[lay.bnd.reshape(-1)] = enc_bits(bbits)
        else:  # trivial words (dataset.hpp:250-253)
            pool[lay.bnd.reshape(-1), K.n] = np.where(bbits == 1, 0x20000000, 0xE0000000)
        sbits = ((b.payload[:, None] >> np.arange(m, dtype=np.uint64)) & 1).astype(np.uint8)
        pool[lay.svc.reshape(-1)] = enc_bits(sbits.reshape(-1))
        ops = W.program_ops(b, lay)
        t = time.perf_counter()
        O.run_program(K, ops, pool, threads, simd="auto")
        dt = time.perf_counter() - t
        got = np.array([sum(O.decrypt_bit(pool[lay.out[q, j]], K.lwe_key) << j for j in range(m))
                        for q in range(Qs)], np.uint64)
        units = b.units()
        full_units = Qfull * Rfull * (12 * l + 2 * m + 3)
        out[name] = {
            "queries_per_s": Qs / dt if Rs == Rfull else (units / dt) / (full_units / Qfull),
            "units_per_s": units / dt, "seconds": dt, "correct": bool(np.array_equal(got, b.truth())),
            "sample": (f"{Qs} query, all {Rfull} boxes, measured" if Rs == Rfull else
                       f"{Qs} query x {Rs} of {Rfull} boxes measured, queries/s extrapolated "
                       f"linearly in bootstrap units"),
        }
    return {"kind": "port", "cores": threads, "unit": "queries/s", "configs": out}


# ---------------------------------------------------------------------------
LOCPIR_SAMPLES = {  # name: queries timed per rank for the flagged modes and --locpir sample
    "cfg1": 1, "cfg3": 1, "cfg4": 256, "cfg5": 32,
}
# queries per program at the stated sizes (each program's scratch: ~19.6 MB per cfg4 query,
# ~154 MB per cfg5 query; every level still spans >= 10 waves of the 148 SMs)
LOCPIR_CHUNK = {"cfg4": 512, "cfg5": 128}
WALL_RESERVE_S = 75.0  # what follows the stated-size runs: flagged samples, batcher, CPU baselines


def run_locpir_suite(args, ctx128, keys128, ws, rank, local, max_over_ranks):
    """LocPIR queries/s for BASELINE.json configs 0, 2, 3, 4 through the batched loc_pir
    program (level-scheduled).  Each rank runs its own shard of queries (cfg4/cfg5:
    queries sharded; cfg1/cfg3: replicas).  Decrypted results are checked against the
    plaintext XOR of the payloads of all containing boxes."""
    import torch
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams, workloads as W
    from paper_2407_19871_b200.dist import GpuBackend, ShardedLocPir
    from paper_2407_19871_b200.engine import plan
    fp64_peak = ctx128.fp64_peak_tflops()
    out = {}
    ctx80 = keys80 = None
    for name, (sec, Qfull, R, l, m, enc) in W.CONFIGS.items():
        if args.locpir_configs and name not in args.locpir_configs.split(","):
            continue
        if sec == 80:
            if ctx80 is None:
                p80 = TfheParams(80)
                keys80 = ClientKeys(p80, KEY_SEED)
                ctx80 = Context(p80, local, stream=torch.cuda.current_stream().cuda_stream)
                ctx80.upload_keys(keys80.bk, keys80.ksk)
            ctx, keys = ctx80, keys80
        else:
            ctx, keys = ctx128, keys128
        be = GpuBackend(ctx, keys, torch.device("cuda", local),
                        staging="host" if BACKEND == "gloo" else "device")
        # flagged modes (not the reference count): "folded" = plaintext-boundary constant
        # folding (plaintext boundaries only), "maj" = majority-borrow
        # comparators (any boundaries)
        # "tree" = log-depth comparators (latency mode, for the single-query cfg1)
        variants = [("", False, False, False)] + \
                   ([("_folded", True, False, False)] if not enc else []) + \
                   ([("_maj", False, True, False)] if name in ("cfg4", "cfg5") else []) + \
                   ([("_tree", True, False, True)] if name == "cfg1" else [])
        for suffix, folded, maj, tree in variants:
            # the reference circuit runs the config at its stated size (all Qfull queries
            # inside the timed region); flagged modes run a labelled per-GPU sample
            full = suffix == "" and args.locpir == "full"
            budget_note = None
            if full and Qfull > LOCPIR_SAMPLES[name]:
                # wall-budget guard: a stated-size run is one timed launch of known length
                # (its bootstraps / the cfg2 gate rate just measured; cfg5 = 26.4 M ~ 250 s).
                # If it would end past --wall-budget (a slower or power-capped box), run the
                # labelled sample instead of overrunning the caller's limit.  The elapsed
                # time is the max over ranks, so every rank takes the same branch.
                est_s = 1.08 * Qfull * R * (12 * l + 2 * m + 3) / ws / max(1.0, args.gate_rate)
                elapsed = max_over_ranks(time.perf_counter() - T_PROCESS)
                if elapsed + est_s + WALL_RESERVE_S > args.wall_budget:
                    full = False
                    budget_note = (f"stated size skipped by --wall-budget {args.wall_budget:.0f} s: "
                                   f"{elapsed:.0f} s elapsed, run predicted {est_s:.0f} s")
            Q = Qfull if full else min(Qfull, LOCPIR_SAMPLES[name])
            # cfg1 replicas (independent queries per GPU); cfg3 boxes sharded
            # (partial XOR roots all-gathered, rank-0 combine level); cfg4/cfg5 queries
            # sharded, results gathered to rank 0 (the stated batch split over the ranks
            # when full, Q queries per rank for a sample).  Every rank builds the same
            # seeded batch.
            if name == "cfg1":
                mode, Qb, bseed, world, rk, scaling = "queries", Q, KEY_SEED + 17 * rank, 1, 0, "replicas"
            elif name == "cfg3":
                mode, Qb, bseed, world, rk, scaling = "boxes", Q, KEY_SEED + 3, ws, rank, "strong"
            elif full:
                mode, Qb, bseed, world, rk, scaling = "queries", Q, KEY_SEED + 4, ws, rank, "strong"
            else:
                mode, Qb, bseed, world, rk, scaling = "queries", Q * ws, KEY_SEED + 4, ws, rank, "weak"
            b = W.make_batch(Qb, R, l, m, seed=bseed, encrypted_bounds=enc)
            for q in range(min(Qb, R)):  # some queries inside boxes
                b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
                b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
            units_ref = b.units()
            if Qb > 64:  # per-query counts from a small batch of the same shape (planning
                small = W.sub_batch(b, 0, 4, 0, R)  # is linear in queries for fixed boxes)
                pl = plan(W.program_ops(small, W.PoolLayout(small), True, folded, maj, tree))
                units = pl["blind_rotations"] // 4 * Qb
            else:
                pl = plan(W.program_ops(b, W.PoolLayout(b), True, folded, maj, tree))
                units = pl["blind_rotations"]
            if full and Qb > 64:
                # stated size: programs of LOCPIR_CHUNK queries sharing one scratch region
                # (every query inside the timed region); warm-up on a small batch of the
                # same shape (kernels, L2 window), then scratch sized before timing -- the
                # full programs' single timed launch enqueues their kernels directly
                wb = W.sub_batch(b, 0, min(Qb, 8 * world), 0, R)
                warm = ShardedLocPir(be, wb, rk, world, mode, seed=5000)
                warm.launch()
                torch.cuda.synchronize()
                warm.close()
                run = ShardedLocPir(be, b, rk, world, mode, seed=5000, folded=folded, maj=maj,
                                    tree=tree, chunk=LOCPIR_CHUNK[name])
                run.prepare()
                reps = 1
            else:
                run = ShardedLocPir(be, b, rk, world, mode, seed=5000, folded=folded, maj=maj,
                                    tree=tree)
                run.launch()  # warm-up
                reps = 3 if units < 200000 else 1
            torch.cuda.synchronize()
            if ws > 1:
                torch.distributed.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                run.launch()
            e1.record()
            torch.cuda.synchronize()
            ms = max_over_ranks(e0.elapsed_time(e1) / reps)
            res = run.results()
            ok = bool(res is None or np.array_equal(res, b.truth()))
            qtot = ws * Qb if scaling == "replicas" else Qb
            out[name + suffix] = {
                "queries_per_s": qtot / (ms / 1e3), "ms_per_batch": ms,
                "queries_per_batch": qtot, "full_batch_queries": Qfull, "boxes": R, "l": l,
                "m": m, "security_bits": sec, "encrypted_boundaries": enc,
                "bootstrap_units_per_query": units // Qb,
                "reference_units_per_query": b.units() // Qb,
                "units_per_s": (qtot // Qb) * units / (ms / 1e3), "correct": ok,
                "sharding": {"cfg1": "replicas", "cfg3": "boxes (partial roots all-gathered, "
                             "rank-0 combine)"}.get(name, "queries (results gathered to rank 0)"),
                "scaling": scaling,
                "levels": pl["levels"],
                "mode": ("flagged: folded log-depth tree comparators, latency mode (not the "
                         "reference gate count)") if tree else
                        ("flagged: plaintext boundaries constant-folded (not the reference "
                         "gate count)") if folded else
                        ("flagged: majority-borrow comparators, N(4l+2m+3)-m units (not the "
                         "reference gate count)") if maj else
                        "reference circuit (N(12l+2m+3) units)",
                "programs": len(run.progs),
                "sample": "full config" if Q == Qfull else f"{Q} of {Qfull} queries per GPU "
                                                           "(per-query cost is batch-independent "
                                                           "once the GPU is saturated)",
                "roofline": locpir_roofline(sec, units / Qb, qtot / (ms / 1e3), ws, fp64_peak),
            }
            if budget_note:
                out[name + suffix]["wall_budget"] = budget_note
            run.close()
    if not args.locpir_configs or "cfg4" in args.locpir_configs.split(","):
        out["cfg4_server"] = run_server_sample(ctx128, keys128, ws, max_over_ranks)
    if ctx80 is not None:  # cfg1's latency roof (single query, 80-bit)
        for key in ("cfg1", "cfg1_tree"):
            if key in out:
                out[key]["latency_roofline"] = latency_floor(ctx80, keys80, out[key]["levels"],
                                                             out[key]["ms_per_batch"])
        ctx80.close()
    if args.emulate_shards and ws == 1:
        out["shard_emulation"] = run_shard_emulation(ctx128, keys128)
    return out


def device_ms(fn, reps=3, warm=True):
    """Mean device time of fn() over reps launches (CUDA events on the current stream)."""
    import torch
    if warm:
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def latency_floor(ctx, keys, levels, measured_ms):
    """cfg1 is latency-bound (a 21-level circuit with <= 68 gates per level): its roof is
    the device time of a chain of `levels` dependent bootstrapped gates (one gate per
    level, the same latency kernels K1l + K2s and the same graph-replayed launch sequence
    as the circuit), i.e. critical-path levels x one level's latency."""
    from paper_2407_19871_b200 import _abi
    ctx.pool_reserve(levels + 2)
    ctx.h2d(0, keys.encrypt_bits(np.array([1, 0], np.uint8), 5))
    chain = [(_abi.NAND, 0, 1, _abi.SLOT_NONE, 2)]
    chain += [(_abi.NAND, 1 + i, 0, _abi.SLOT_NONE, 2 + i) for i in range(1, levels)]
    prog = ctx.program(chain)
    t_chain = device_ms(prog.launch, reps=5)
    prog.close()
    return {"bound": "latency", "levels": levels, "one_gate_ms": t_chain / levels,
            "floor_ms": t_chain, "measured_ms": measured_ms, "frac": t_chain / measured_ms,
            "note": "floor = device time of a chain of `levels` dependent bootstrapped gates "
                    "(critical-path levels x one level's latency)"}


def run_shard_emulation(ctx, keys, Ns=(2, 4, 8)):
    """--emulate-shards: the N-GPU LocPIR shards run one after another on
    this one GPU.  cfg3 (box-sharded, strong scaling): every rank's box shard is evaluated
    (xor_tree mode 2), the partial roots are copied into the rank-0 combine region and the
    combine level runs; predicted N-GPU time = max shard time + combine time (the gather of
    N x 32 ciphertexts over NVLink is ~us and not modelled).  cfg4/cfg5 (query-sharded):
    the largest shard (Q/N queries) is timed; predicted time = that shard's time.  Results
    are decrypted and checked against the plaintext truth."""
    import torch
    from paper_2407_19871_b200 import workloads as W
    from paper_2407_19871_b200.dist import shard_range
    out = {}
    sec, Q, R, l, m, enc = W.CONFIGS["cfg3"]
    b = W.make_batch(Q, R, l, m, seed=KEY_SEED + 3, encrypted_bounds=enc)
    b.x[0] = (b.boxes[0, 0] + b.boxes[0, 1]) // 2
    b.y[0] = (b.boxes[0, 2] + b.boxes[0, 3]) // 2
    n1 = ctx.params.n + 1
    rows = {}
    for N in Ns:
        spans = [shard_range(R, r, N) for r in range(N)]
        t_shards, parts = [], []
        for lo, hi in spans:
            sub = W.sub_batch(b, 0, Q, lo, hi)
            lay = W.PoolLayout(sub)
            ctx.pool_reserve(lay.total)
            W.load_batch(ctx, keys, sub, lay, 5000 + lo)
            prog = ctx.program(W.program_ops(sub, lay, 2))
            t_shards.append(device_ms(prog.launch, reps=1))
            parts.append(ctx.d2h(int(lay.out.min()), Q * m))
            prog.close()
        part_first, out_first = 0, N * Q * m
        comb_first = out_first + Q * m
        ctx.pool_reserve(comb_first + Q * m * (N + 1))
        ctx.h2d(part_first, np.concatenate(parts))
        comb = ctx.program(W.combine_ops(N, Q, m, part_first, out_first, comb_first))
        t_comb = device_ms(comb.launch, reps=1)
        comb.close()
        bits = keys.decrypt_bits(ctx.d2h(out_first, Q * m)).reshape(Q, m).astype(np.uint64)
        got = (bits << np.arange(m, dtype=np.uint64)).sum(axis=1)
        t = max(t_shards) + t_comb
        rows[N] = {"boxes_per_gpu": spans[0][1] - spans[0][0], "max_shard_ms": max(t_shards),
                   "combine_ms": t_comb, "predicted_ms": t, "predicted_queries_per_s": Q / (t / 1e3),
                   "correct": bool(np.array_equal(got, b.truth()))}
    out["cfg3"] = {"sharding": "boxes (strong scaling)", "per_N": rows}
    for name in ("cfg4", "cfg5"):
        sec, Q, R, l, m, enc = W.CONFIGS[name]
        rows = {}
        for N in Ns[-1:]:
            lo, hi = shard_range(Q, 0, N)
            b = W.make_batch(hi - lo, R, l, m, seed=KEY_SEED + 4, encrypted_bounds=enc)
            for q in range(min(hi - lo, R)):
                b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
                b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
            lay = W.PoolLayout(b, LOCPIR_CHUNK[name])
            ctx.pool_reserve(lay.total)
            W.load_batch(ctx, keys, b, lay, 5000)
            progs = [ctx.program(W.program_ops(b, lay, True, q_lo=a, q_hi=z)) for a, z in lay.chunks()]
            for p_ in progs:
                p_.prepare()
            t = device_ms(lambda: [p_.launch() for p_ in progs], reps=1, warm=False)
            bits = keys.decrypt_bits(ctx.d2h(int(lay.out.min()), b.Q * m)).reshape(b.Q, m)
            got = (bits.astype(np.uint64) << np.arange(m, dtype=np.uint64)).sum(axis=1)
            for p_ in progs:
                p_.close()
            rows[N] = {"queries_per_gpu": hi - lo, "shard_ms": t,
                       "predicted_queries_per_s": Q / (t / 1e3),
                       "correct": bool(np.array_equal(got, b.truth()))}
        out[name] = {"sharding": "queries (strong scaling of the stated batch)", "per_N": rows}
    out["label"] = ("single-GPU emulation of the N-GPU shards (no multi-GPU box was "
                    "available); not a measured multi-GPU number")
    return out


def run_server_sample(ctx, keys, ws, max_over_ranks, Q=256, sessions=8):
    """cfg4's shape through the cross-session batcher: QUERY payload bytes
    of `sessions` sessions in, RESPONSE bytes out.  The timed region holds submit (framing
    checks), flush (one H2D of all payloads + unpack, planning, the batched program,
    response pack + one D2H) and take_response; sessions' zero sheets are registered
    before it.  Replicas per GPU."""
    import torch
    from paper_2407_19871_b200 import workloads as W
    from paper_2407_19871_b200.server import BatchingServer
    sec, _, R, l, m, _ = W.CONFIGS["cfg4"]
    b = W.make_batch(Q, R, l, m, seed=KEY_SEED + 9)
    for q in range(min(Q, R)):
        b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    srv = BatchingServer(ctx, W.signed_boxes(b), b.payload, l, m, max_sessions=sessions)
    n1 = ctx.params.n + 1
    # client side (untimed): zero sheets = Enc(-1/8) + 1/8 = Enc(0); framed query words
    sids = []
    for s_ in range(sessions):
        z = keys.encrypt_bits(np.zeros(R * m, np.uint8), 7000 + s_)
        z[:, -1] += np.uint32(0x20000000)
        sids.append(srv.open_session(z.astype("<u4").tobytes()))
    xb = W._bits_signed(b.x, l)
    yb = W._bits_signed(b.y, l)
    cx = keys.encrypt_bits(xb.reshape(-1), 8000).reshape(Q, l, n1)
    cy = keys.encrypt_bits(yb.reshape(-1), 8001).reshape(Q, l, n1)
    payloads = [bytes([l]) + cx[q].astype("<u4").tobytes() + bytes([l]) + cy[q].astype("<u4").tobytes()
                for q in range(Q)]

    def one_round():
        tickets = [srv.submit(sids[q % sessions], payloads[q]) for q in range(Q)]
        srv.flush()
        return [srv.take_response(t) for t in tickets]

    one_round()  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    resp = one_round()
    dt = max_over_ranks(time.perf_counter() - t0)
    got = np.array([(keys.decrypt_bits(np.frombuffer(r, "<u4").reshape(m, n1)).astype(np.uint64)
                     << np.arange(m, dtype=np.uint64)).sum() for r in resp], np.uint64)
    srv.close()
    return {"queries_per_s": ws * Q / dt, "ms_per_batch": dt * 1e3, "queries_per_gpu": Q,
            "sessions": sessions, "boxes": R, "l": l, "m": m, "security_bits": sec,
            "correct": bool(np.array_equal(got, b.truth())),
            "h2d_bytes_per_batch": sum(len(p_) for p_ in payloads),
            "d2h_bytes_per_batch": Q * m * 4 * n1,
            "mode": "wire path: QUERY bytes -> batched loc_pir -> RESPONSE bytes (host clock, "
                    "includes payload copies, framing checks and planning)"}


# ---------------------------------------------------------------------------
# LOCPIR_BENCH_BACKEND=gloo (tests only): N ranks sharing fewer GPUs exchange through host
# memory; the timing is then not a multi-GPU measurement, the code path is the N > 1 one
BACKEND = os.environ.get("LOCPIR_BENCH_BACKEND", "nccl")


def run_b200(args):
    import torch
    ws, rank, local = dist_env()
    if BACKEND == "gloo":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if BACKEND == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams, _abi

    params = TfheParams(SECURITY)
    stream = torch.cuda.Stream()  # a real stream handle: the library launches on it and the
    torch.cuda.set_stream(stream)  # CUDA events below are recorded on the same stream
    ctx = Context(params, local, stream=stream.cuda_stream)
    G = args.gates
    n1 = params.n + 1

    # ---- keys: generated once (client side) and broadcast over NVLink to every GPU
    from paper_2407_19871_b200.dist import broadcast_keys, max_over_ranks as _mor
    t_setup = time.perf_counter()
    keys, bk_t, ksk_t = broadcast_keys(params, KEY_SEED, rank,
                                       device=None if BACKEND == "gloo" else "cuda")
    torch.cuda.synchronize()
    if BACKEND == "gloo":
        ctx.upload_keys(bk_t.numpy().view(np.uint32), ksk_t.numpy().view(np.uint32))
    else:
        ctx.upload_keys(bk_t.data_ptr(), ksk_t.data_ptr(), on_device=True)
    del bk_t, ksk_t

    # ---- this rank's shard of seeded inputs (client-side encryption)
    rng = np.random.default_rng(KEY_SEED + rank)
    A = rng.integers(0, 2, G).astype(np.uint8)
    B = rng.integers(0, 2, G).astype(np.uint8)
    a = keys.encrypt_bits(A, 1000 + 2 * rank)
    b = keys.encrypt_bits(B, 1001 + 2 * rank)
    ctx.pool_reserve(3 * G)
    ctx.h2d(0, a)
    ctx.h2d(G, b)
    prog = ctx.program([(_abi.NAND, g, G + g, _abi.SLOT_NONE, 2 * G + g) for g in range(G)])
    setup_s = time.perf_counter() - t_setup

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        return _mor(x, device=None if BACKEND == "gloo" else "cuda")

    # ---- device-resident throughput (value)
    for _ in range(args.warmup):
        prog.launch()
    torch.cuda.synchronize()
    out = ctx.d2h(2 * G, G)
    correct = bool(np.array_equal(keys.decrypt_bits(out), 1 - (A & B)))

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ctx.timing(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        prog.launch()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    stats = ctx.kernel_stats()
    ctx.timing(False)
    barrier()
    ms_step = ms_total / args.steps
    value = ws * G / (ms_step / 1000.0)

    # ---- roofline of the dominant kernel (K1 blind rotate), measured live
    br_ms, br_launches = stats["blind_rotate"]
    ks_ms, ks_launches = stats["keyswitch"]
    avg_br_ms = br_ms / max(1, br_launches)
    achieved_tflops = G * flop_per_br() / (avg_br_ms * 1e-3) / 1e12
    peak = ctx.fp64_peak_tflops()
    ksk_bytes = params.ksk_words() * 4
    avg_ks_ms = ks_ms / max(1, ks_launches)

    # ---- end to end through the C ABI with pinned host buffers
    a_h = torch.from_numpy(a).pin_memory()
    b_h = torch.from_numpy(b).pin_memory()
    o_h = torch.empty((G, n1), dtype=torch.int32).pin_memory()
    ctx.gate_batch_host_ptr(_abi.NAND, a_h.data_ptr(), b_h.data_ptr(), o_h.data_ptr(), G)
    e2e_steps = max(1, args.steps)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ctx.gate_batch_host_ptr(_abi.NAND, a_h.data_ptr(), b_h.data_ptr(), o_h.data_ptr(), G)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e_ok = bool(np.array_equal(keys.decrypt_bits(o_h.numpy().view(np.uint32)), 1 - (A & B)))

    args.gate_rate = value / ws  # per-GPU bootstraps/s, for the wall-budget guard
    locpir_results = None if args.no_locpir else run_locpir_suite(args, ctx, keys, ws, rank,
                                                                   local, max_over_ranks)
    if rank == 0:
        line = {
            "metric": "bootstrapped gates/s (128-bit TFHE)", "value": value, "unit": "gates/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded uniform bits encrypted under seeded keys",
            "config": workload_config(ws),
            "correct": correct and e2e_ok,
            "roofline": {
                "bound": "fp64", "kernel": "k_blind_rotate<3,7> (K1)",
                "achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved_tflops / peak if peak else None,
                "traffic": committed_traffic() if G == GATES_PER_GPU else None,
                "traffic_unit": "bytes per launch (DRAM read+write, the newest ncu capture "
                                "in profiles/r0N_traffic.json)",
                "algorithmic_bytes_per_launch": G * (2 * 4 * (params.n + 1) + 4 * (params.N + 1))
                                                + params.bk_words() * 8,
                "flop_per_unit": flop_per_br(), "units_per_launch": G,
                "avg_launch_ms": avg_br_ms,
                "peak_source": "measured live on this GPU: k_fp64_peak DFMA microbenchmark "
                               "(MEASURED_PEAKS.json has no FP64 figure)",
                "step_share": br_ms / max(1e-9, br_ms + ks_ms),
                "bound_note": "FP64 pipe: per-ciphertext negacyclic FFTs are dense FP64 work "
                              "with no shared contraction (SURVEY §8(d)), so neither the HBM "
                              "nor the tensor-core roof applies; hbm_view shows the HBM side",
                "hbm_view": hbm_view(G, params, avg_br_ms),
                "l1tex_view": l1tex_view(),
            },
            "keyswitch": keyswitch_view(G, params, avg_ks_ms, ksk_bytes),
            "e2e": {"value": ws * G / e2e_s, "unit": "gates/s",
                    "h2d_bytes_per_step": 2 * G * n1 * 4, "d2h_bytes_per_step": G * n1 * 4,
                    "path": "locpir_b200_gate_batch_host on pinned host buffers: the input rows "
                            "cross PCIe inside the blind rotation's prologue (zero-copy reads "
                            "of the caller's buffers), the outputs are packed and copied back "
                            "before the call returns"},
            "gpu_launches": args.steps * prog.kernels,
            "clocks": clk,
            "setup_s": setup_s,
        }
        if not args.no_locpir:
            line["locpir"] = locpir_results
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_oracle_rate(budget_s=args.ref_budget)
            line["cpu_baseline"]["host_cpu"] = host_cpu()
            line["reference_standin"] = standin_rate()
            if not args.no_locpir:
                line["cpu_baseline_locpir"] = cpu_locpir_baseline()
                line["reference_standin_locpir"] = standin_locpir_rates()
        print(json.dumps(line), flush=True)
    prog.close()
    ctx.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def spawn_ranks(n):
    """`bench.py --gpus N` (N > 1) started as a plain process: re-launch this command as N
    ranks, one process per GPU, the way the driver does (torch.distributed.run, rendezvous
    on 127.0.0.1).  NCCL_DEBUG=INFO keeps NCCL's communicator lines (nranks) in stderr."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def run_dry(args):
    """--dry-run (no GPU needed): the multi-rank plumbing of the bench -- rank spawn, gloo
    process group, query sharding of a small cfg4-shaped batch, the gather to rank 0,
    barrier-bracketed timing and the max over ranks -- with the plaintext interpreter of
    tests/plain_backend.py (test infrastructure) standing in for each rank's GPU."""
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from plain_backend import PlainBackend
    from paper_2407_19871_b200 import workloads as W
    from paper_2407_19871_b200.dist import ShardedLocPir, max_over_ranks
    sec, _, R, l, m, _ = W.CONFIGS["cfg4"]
    Q = 8 * ws
    b = W.make_batch(Q, R, l, m, seed=KEY_SEED + 4)
    for q in range(min(Q, R)):
        b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    run = ShardedLocPir(PlainBackend(), b, rank, ws, "queries", seed=5)
    for _ in range(args.warmup):
        run.launch()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run.launch()
    if ws > 1:
        dist.barrier()
    dt = max_over_ranks((time.perf_counter() - t0) / args.steps)
    res = run.results()
    if rank == 0:
        print(json.dumps({
            "dry_run": True, "metric": "LocPIR queries/s (plaintext interpreter, plumbing only)",
            "value": Q / dt, "unit": "queries/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "correct": bool(np.array_equal(res, b.truth())),
            "config": {"workload": f"cfg4 shape, {Q} queries x {R} boxes, queries sharded",
                       "backend": "gloo"}}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


ORACLE_BUILD = "x86-64-v3"


def select_oracle_build():
    """The CPU baseline uses the AVX-512 build of the oracle port when the host has it
    (bit-identical results: -ffp-contract=off, no fast-math)."""
    global ORACLE_BUILD
    v4 = os.path.join(ROOT, "oracle", "build", "liboracle_v4.so")
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        flags = ""
    if " avx512f" in flags and os.path.exists(v4) and "LOCPIR_ORACLE_LIB" not in os.environ:
        os.environ["LOCPIR_ORACLE_LIB"] = v4
        ORACLE_BUILD = "x86-64-v4 (AVX-512)"


def main():
    select_oracle_build()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--ref-budget", type=float, default=12.0,
                    help="seconds of CPU work per reference/cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-locpir", action="store_true",
                    help="skip the LocPIR queries/s measurements (configs 0, 2, 3, 4)")
    ap.add_argument("--locpir", default="full", choices=["full", "sample"],
                    help="full: cfg4/cfg5 reference circuits at their stated sizes (default); "
                         "sample: LOCPIR_SAMPLES queries per GPU (quick runs)")
    ap.add_argument("--wall-budget", type=float, default=720.0,
                    help="seconds of wall time the whole run may take: a stated-size LocPIR run "
                         "predicted to end later falls back to its labelled sample (a default "
                         "run takes ~8 min on a B200 at full clocks)")
    ap.add_argument("--gates", type=int, default=GATES_PER_GPU,
                    help="gates per GPU (default: the cfg2 size; smaller only for profiling)")
    ap.add_argument("--locpir-configs", default="",
                    help="comma-separated subset of cfg1,cfg3,cfg4,cfg5 (default: all)")
    ap.add_argument("--emulate-shards", action="store_true",
                    help="also run the N = 2/4/8 LocPIR shards one after another on this GPU")
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank plumbing only (gloo, plaintext interpreter, no GPU)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
