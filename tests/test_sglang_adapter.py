"""The SGLang-style adapter (sglang_adapter.py): match_prefix returns the pool
rows of the cached prefix, insert writes the new tokens' KV into their rows,
evict returns rows to the pool, locks protect prefixes -- and hits / victims
equal the reference semantics (the oracle cache driven with the same ops)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BPT = 32


def _kv(tokens, pos):
    x = np.asarray(tokens, np.uint64) * np.uint64(0x9E3779B97F4A7C15) + np.asarray(pos, np.uint64)
    return np.stack([x, x ^ np.uint64(0xABCDEF), x + np.uint64(7), x * np.uint64(3)], axis=1).view(np.uint8)


def test_sglang_adapter_ops():
    import torch

    from oracle.oracle import OracleRadixCache
    from paper_2605_08581_b200.sglang_adapter import SGLangRadixCache
    from paper_2605_08581_b200.types import CacheConfig, CachePolicy

    rng = np.random.default_rng(0)
    cap = 5000
    ad = SGLangRadixCache(cap, BPT)
    ora = OracleRadixCache(CacheConfig(capacity_tokens=cap, policy=CachePolicy.LRU, protect_budget=0))
    prompts = [[int(x) for x in rng.integers(0, 50, size=int(rng.integers(20, 400)))] for _ in range(12)]
    for step in range(150):
        base = prompts[int(rng.integers(0, len(prompts)))]
        key = base[:int(rng.integers(1, len(base) + 1))] + [int(x) for x in rng.integers(100, 10**6, size=int(rng.integers(0, 60)))]
        rows, last = ad.match_prefix(key)
        hit = ora.match_prefix(key)[0]
        assert rows.shape[0] == hit, step
        if hit:  # the cached prefix's rows hold the KV written when it was inserted
            pool = torch.zeros((hit, BPT), dtype=torch.uint8, device="cuda")
            got = ad.kv.gather(torch.tensor([last.slot], dtype=torch.int32, device="cuda"), 1, hit, payload=True)[2]
            assert np.array_equal(got[0, :hit].cpu().numpy(), _kv(key[:hit], np.arange(hit))), step
        new = _kv(key[hit:], np.arange(hit, len(key)))
        try:
            prefix = ad.insert(key, torch.from_numpy(np.ascontiguousarray(new)).cuda() if len(new) else None)
        except Exception as e:  # CapacityError: everything else is locked
            assert "CapacityError" in type(e).__name__
            continue
        assert prefix == hit
        leaf = ora.insert_path(key)
        ora.release_path(leaf)
        if rng.random() < 0.1:
            k = int(rng.integers(0, 2000))
            assert ad.evict(k) == ora.evict(k)
        st = ad.kv_stats()
        assert st["rows"] - st["free"] == ad.total_size() == ora.resident_tokens
        assert ad.evictable_size() + ad.protected_size() == ad.total_size()
    assert ad.cache.victim_log() == ora.victim_log()
    ad.close()


def test_sglang_adapter_locks():
    """A locked prefix survives any eviction (its tokens are the protected
    size); unlocking makes it evictable again and its rows return to the pool."""
    import torch

    from paper_2605_08581_b200.sglang_adapter import SGLangRadixCache

    ad = SGLangRadixCache(10_000, BPT)
    a, b = list(range(1000, 1300)), list(range(5000, 5200))
    ad.insert(a)
    ad.insert(b)
    rows, node = ad.match_prefix(a)
    assert rows.shape[0] == 300 and ad.protected_size() == 0
    ad.inc_lock_ref(node)
    assert ad.protected_size() == 300
    assert ad.evict(10_000) == 200  # only b goes
    assert ad.total_size() == 300 and ad.match_prefix(a)[0].shape[0] == 300
    assert ad.match_prefix(b)[0].shape[0] == 0
    ad.dec_lock_ref(node)
    assert ad.protected_size() == 0 and ad.evict(10_000) == 300
    st = ad.kv_stats()
    assert ad.total_size() == 0 and st["free"] == st["rows"]
    with pytest.raises(ValueError):
        ad.dec_lock_ref(node)
    ad.close()
