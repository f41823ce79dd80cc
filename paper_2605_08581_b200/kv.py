"""Paged KV payload behind a device tree (csrc/kv.cuh; north_star item 4).

``KvPool(tree_handle, rows, bytes_per_token)`` gives every resident token of
the tree a row of a KV pool in HBM.  After tree operations (a fused wave, a
per-call insert / evict) ``sync(src, dst)`` allocates rows for the newly
resident tokens (in admission order -- each admitted request's uncached
tokens; ``src`` holds their KV in that order) and returns the victims' rows to
the free stack (``dst`` receives their KV in eviction order).  ``gather``
builds a request's ``req_to_token`` row table from its leaf and optionally
copies the KV rows out.  All buffers are torch CUDA tensors (plumbing only).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check

_p, _i64 = C.c_void_p, C.c_int64


def _bind(L):
    for name, res, args in (("prism_kv_enable", C.c_int, [_p, _i64, _i64]),
                            ("prism_kv_sync", C.c_int, [_p, _p, _p, _p]),
                            ("prism_kv_gather", C.c_int, [_p, _i64, _p, _i64, _p, _p, _p]),
                            ("prism_kv_stats", C.c_int, [_p, _p])):
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    return L


class KvPool:
    def __init__(self, tree_handle, rows: int, bytes_per_token: int):
        self.L = _bind(_lib.lib())
        self.h = tree_handle
        self.rows, self.bpt = int(rows), int(bytes_per_token)
        check(self.L.prism_kv_enable(self.h, self.rows, self.bpt))

    def sync(self, src: torch.Tensor | None = None, dst: torch.Tensor | None = None,
             counts: bool = True) -> tuple[int, int] | None:
        """(new resident tokens, freed tokens) since the last sync.  ``src``:
        uint8 [>= new, bytes_per_token] of the new tokens' KV (admission
        order); ``dst``: uint8 [>= freed, bytes_per_token] for the victims' KV.
        ``counts=False``: no host wait (the work stays queued on the tree's stream)."""
        out = np.zeros(2, np.int64)
        for t in (src, dst):  # (produced on torch's stream; the pool works on the tree's)
            if t is not None:
                torch.cuda.current_stream(t.device).synchronize()
        check(self.L.prism_kv_sync(self.h, src.data_ptr() if src is not None else None,
                                   dst.data_ptr() if dst is not None else None,
                                   out.ctypes.data if counts else None))
        return (int(out[0]), int(out[1])) if counts else None

    def gather(self, leaf_slots: torch.Tensor, n: int, max_len: int, payload: bool = False, wait: bool = True):
        """(table int32 [n, max_len], lens int64 [n], kv uint8 [n, max_len, bpt] or None)."""
        dev = leaf_slots.device
        table = torch.full((max(n, 1), max_len), -1, dtype=torch.int32, device=dev)
        lens = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
        out = torch.zeros((max(n, 1), max_len, self.bpt), dtype=torch.uint8, device=dev) if payload else None
        torch.cuda.current_stream(dev).synchronize()  # (the fills above and leaf_slots: torch's stream)
        check(self.L.prism_kv_gather(self.h, n, leaf_slots.data_ptr(), max_len, table.data_ptr(),
                                     out.data_ptr() if out is not None else None, lens.data_ptr()))
        if wait:  # (the gather runs on the tree's stream)
            self.L.prism_tree_stream.restype = C.c_void_p
            self.L.prism_tree_stream.argtypes = [_p]
            torch.cuda.ExternalStream(self.L.prism_tree_stream(self.h), device=dev).synchronize()
        return table[:n], lens[:n], (out[:n] if out is not None else None)

    def stats(self) -> dict:
        out = np.zeros(6, np.int64)
        check(self.L.prism_kv_stats(self.h, out.ctypes.data))
        return dict(zip(("free", "rows", "allocated", "freed", "bytes_in", "bytes_out"), out.tolist()))
