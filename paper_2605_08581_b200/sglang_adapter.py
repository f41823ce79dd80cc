"""SGLang-style prefix cache over the device DART tree.

The paper integrates PRISM into SGLang's RadixCache; that source is not part
of the reference, so this adapter follows the public shape of SGLang's cache
interface -- ``match_prefix(key) -> (kv indices, last node)``,
``insert(key, value)``, ``evict(num_tokens)``, ``inc_lock_ref / dec_lock_ref``,
``evictable_size / protected_size / total_size`` -- over this package's own
tree (reference semantics: kvcache.py) and its paged KV payload (kv.cuh):
the "KV indices" of a cached prefix are the pool rows of its tokens
(``req_to_token``), and the KV rows of evicted tokens go back to the pool's
free stack.  Parity is pinned against the reference cache's semantics (the
same operations on the oracle give the same hits and victims), not against
SGLang itself (unpinned: no SGLang source in the reference).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from ._lib import check
from .dart import DeviceNode, DeviceRadixCache
from .kv import KvPool
from .types import CacheConfig, CachePolicy


class SGLangRadixCache:
    """``SGLangRadixCache(capacity_tokens, kv_bytes_per_token)``: LRU eviction by
    default (SGLang's), any reference policy accepted."""

    def __init__(self, capacity_tokens: int, kv_bytes_per_token: int = 64, policy=CachePolicy.LRU,
                 device: int = 0, kv_rows: int = 0):
        self.cache = DeviceRadixCache(CacheConfig(capacity_tokens=capacity_tokens, policy=policy, protect_budget=0),
                                      device=device)
        self.kv = KvPool(self.cache._h, kv_rows or 2 * capacity_tokens, kv_bytes_per_token)
        self.dev = torch.device("cuda", device)
        self._locks: dict[int, int] = {}  # slot -> explicit locks taken through this adapter

    # ------------------------------------------------------------ lookups
    def match_prefix(self, key: Sequence[int]) -> tuple[torch.Tensor, DeviceNode | None]:
        """(pool rows of the longest cached prefix, int32 on the device; its
        deepest node or None) -- match_prefix (kvcache.py:146-171) refreshes
        the visited nodes' recency like SGLang's access-time update."""
        hit, nodes = self.cache.match_prefix(key)
        if hit == 0 or not nodes:
            return torch.zeros(0, dtype=torch.int32, device=self.dev), None
        last = nodes[-1]
        # (positions past the key -- a match ending inside a node -- are not written)
        table, _, _ = self.kv.gather(torch.tensor([last.slot], dtype=torch.int32, device=self.dev), 1, hit)
        return table[0, :hit].clone(), last

    def insert(self, key: Sequence[int], value: torch.Tensor | None = None) -> int:
        """Cache ``key``; returns the length of the prefix that was already
        cached.  ``value`` (uint8 [len(key) - prefix, bytes_per_token], device)
        is the KV of the new tokens, written into their pool rows.  May evict
        (the reference's _reserve, kvcache.py:243-273)."""
        hit = self.cache.match_prefix(key)[0]
        leaf = self.cache.insert_path(key)
        self.cache.release_path(leaf)  # SGLang's insert takes no lock
        self.kv.sync(value)
        return hit

    def evict(self, num_tokens: int) -> int:
        """Free at least num_tokens tokens (kvcache.py:425-460); their KV rows
        return to the pool.  Returns the tokens freed."""
        freed = self.cache.evict(int(num_tokens))
        self.kv.sync()
        return freed

    # ------------------------------------------------------------ locks
    def inc_lock_ref(self, node: DeviceNode | None) -> None:
        if node is None:
            return
        s = torch.tensor([node.slot], dtype=torch.int32, device=self.dev)
        torch.cuda.current_stream(self.dev).synchronize()  # (the slot's copy runs on torch's stream)
        check(self.cache._L.prism_pin_device(self.cache._h, 1, s.data_ptr(), None))
        torch.cuda.synchronize(self.dev)
        self._locks[node.slot] = self._locks.get(node.slot, 0) + 1
        self.cache._dirty()

    def dec_lock_ref(self, node: DeviceNode | None) -> None:
        if node is None:
            return
        if self._locks.get(node.slot, 0) <= 0:
            raise ValueError("dec_lock_ref without a matching inc_lock_ref")
        self.cache.release_path(node)
        self._locks[node.slot] -= 1

    # ------------------------------------------------------------ sizes
    def total_size(self) -> int:
        return self.cache.resident_tokens

    def protected_size(self) -> int:
        """Tokens of locked nodes (ref > 0)."""
        s = self.cache._snapshot()
        live = (s["nid"] >= 0) & (s["par"] >= 0)
        live[0] = False
        return int(s["elen"][live & (s["ref"] > 0)].sum())

    def evictable_size(self) -> int:
        return self.total_size() - self.protected_size()

    def kv_stats(self) -> dict:
        return self.kv.stats()

    def close(self) -> None:
        self.cache.close()
