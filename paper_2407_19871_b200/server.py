"""Cross-session LocPIR query batcher -- Python face of
locpir_b200_server_* (csrc/server.hpp).  Mirrors Server::handle_zerosheet /
handle_query (protocol.hpp:373-424) minus the transport: wire payloads in, wire payloads
out, every flush one batched program over all sessions' pending queries."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import lib
from .engine import InvalidArgument, LogicError


class BatchingServer:
    def __init__(self, ctx, boxes, services, l: int, m: int, max_sessions: int = 64,
                 folded: bool = False, base_slot: int = 0):
        """boxes: [R, 4] signed l-bit grid values (x1, x2, y1, y2); services: [R] values.
        The server owns every pool slot from base_slot on (0: a dedicated context); other
        calls on the context that touch those slots fail (include/locpir_b200.h)."""
        self.ctx, self.l, self.m = ctx, l, m
        bx = np.ascontiguousarray(boxes, np.int64).reshape(-1, 4)
        sv = np.ascontiguousarray(services, np.uint64).reshape(-1)
        if sv.size != bx.shape[0]:
            raise InvalidArgument("one service value per box")
        h = C.c_void_p()
        rc = lib().locpir_b200_server_create_at(ctx.h, base_slot,
                                                bx.ctypes.data_as(C.POINTER(C.c_int64)),
                                                sv.ctypes.data_as(C.POINTER(C.c_uint64)),
                                                bx.shape[0], l, m, max_sessions, int(folded),
                                                C.byref(h))
        if rc:
            raise InvalidArgument(lib().locpir_b200_last_error(ctx.h).decode())
        self.h = h
        self.response_bytes = m * 4 * (ctx.params.n + 1)

    def _c(self, rc):
        if rc == _abi.OK:
            return
        msg = lib().locpir_b200_server_last_error(self.h).decode()
        if rc == _abi.EINVAL:
            raise InvalidArgument(msg)
        if rc == _abi.ELOGIC:
            raise LogicError(msg)
        raise RuntimeError(msg)

    def open_session(self, zero_sheet: bytes) -> int:
        sid = C.c_uint32()
        raw = np.frombuffer(zero_sheet, np.uint8) if zero_sheet else np.zeros(1, np.uint8)
        self._c(lib().locpir_b200_server_open_session(self.h, raw.ctypes.data, len(zero_sheet),
                                                      C.byref(sid)))
        return sid.value

    def close_session(self, sid: int):
        self._c(lib().locpir_b200_server_close_session(self.h, sid))

    def submit(self, sid: int, query: bytes) -> int:
        t = C.c_uint64()
        raw = np.frombuffer(query, np.uint8) if query else np.zeros(1, np.uint8)
        self._c(lib().locpir_b200_server_submit(self.h, sid, raw.ctypes.data, len(query),
                                                C.byref(t)))
        return t.value

    @property
    def pending(self) -> int:
        return lib().locpir_b200_server_pending(self.h)

    def flush(self) -> int:
        n = C.c_uint64()
        self._c(lib().locpir_b200_server_flush(self.h, C.byref(n)))
        return n.value

    def take_response(self, ticket: int) -> bytes:
        out = np.zeros(self.response_bytes, np.uint8)
        self._c(lib().locpir_b200_server_take_response(self.h, ticket, out.ctypes.data, out.size))
        return out.tobytes()

    def close(self):
        if getattr(self, "h", None):
            lib().locpir_b200_server_destroy(self.h)
            self.h = None

    def __del__(self):
        try:  # interpreter shutdown may already have torn down the module globals
            self.close()
        except Exception:
            pass
