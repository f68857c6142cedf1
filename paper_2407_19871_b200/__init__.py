"""B200-native TFHE gate bootstrapping for LocPIR (arxiv 2407.19871).

Drop-in for the reference engine boundary (gate_engine.hpp:130-336): the
bootstrapped gates, the comparator and the LocPIR query evaluator run as
hand-written sm_100a kernels behind the C ABI in include/locpir_b200.h.
Importing the package loads the in-tree CUDA library and fails loudly if it
is missing -- there is no CPU fallback.
"""
from ._abi import lib as _lib

_lib()  # fail loudly at import when the CUDA extension is absent

from .engine import (ClientKeys, CipherBit, Context, GateEngine, InvalidArgument,  # noqa: E402
                     LogicError, TfheParams, check_query_payload, loc_pir_folded_program,
                     loc_pir_program, loc_pir_program_ex, parse_engine_kind, plan)
from .server import BatchingServer  # noqa: E402
from . import circuits, workloads  # noqa: E402,F401

__all__ = ["ClientKeys", "CipherBit", "Context", "GateEngine", "InvalidArgument", "LogicError",
           "TfheParams", "BatchingServer", "check_query_payload", "loc_pir_program",
           "loc_pir_program_ex", "loc_pir_folded_program", "parse_engine_kind", "plan",
           "circuits", "workloads"]
