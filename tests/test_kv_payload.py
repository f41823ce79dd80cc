"""The paged KV payload (csrc/kv.cuh) behind the device tree.

Every resident token owns a pool row; the parity-checkable parts of the
reference (token-granular, no payload) are the token counts: rows in use ==
resident tokens after every sync, rows freed == the victims' tokens.  The
payload itself is checked by construction: the KV written for a token is a
function of (token, path position) -- identical prefixes have identical
(token, position) pairs -- so every gathered row of every pinned request must
equal f(token, position), whichever earlier request (or wave) wrote it.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BPT = 64


def _rows(tokens: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """f(token, position): BPT bytes per token."""
    x = (tokens.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15) + pos.astype(np.uint64) * np.uint64(0xC2B2AE35))
    words = np.stack([x ^ np.uint64(k * 0x100000001B3) for k in range(BPT // 8)], axis=1)
    return words.view(np.uint8).reshape(len(tokens), BPT)


@pytest.mark.parametrize("seed", range(3))
def test_per_call_payload(seed):
    import torch

    from oracle.oracle import OracleRadixCache
    from paper_2605_08581_b200.dart import DeviceRadixCache
    from paper_2605_08581_b200.kv import KvPool
    from paper_2605_08581_b200.types import Anchor, CacheConfig, CachePolicy, CapacityError, NodeKind

    rng = np.random.default_rng(seed)
    cap = 3000
    cfg = CacheConfig(capacity_tokens=cap, policy=CachePolicy.LRU, protect_budget=0)
    dev, ora = DeviceRadixCache(cfg), OracleRadixCache(cfg)
    kv = KvPool(dev._h, 2 * cap, BPT)
    pinned, opaths = [], {}
    for step in range(60):
        batch_src, nb = [], 0
        for _ in range(int(rng.integers(1, 5))):
            L = int(rng.integers(5, 200))
            base = int(rng.integers(0, 6))
            path = [base * 1000 + i for i in range(L // 2)] + [int(x) for x in rng.integers(0, 10**6, size=L - L // 2)]
            anchors = [Anchor(int(rng.integers(1, L)), NodeKind.REUSABLE, int(rng.integers(0, 9)))]
            hit = dev.match_prefix(path)[0]
            assert hit == ora.match_prefix(path)[0]
            try:
                leaf = dev.insert_path(path, anchors)
            except CapacityError:
                with pytest.raises(CapacityError):
                    ora.insert_path(path, anchors)
                continue
            oleaf = ora.insert_path(path, anchors)
            p = np.array(path, np.uint32)
            batch_src.append(_rows(p[hit:], np.arange(hit, len(p))))
            pinned.append((leaf, oleaf, p))
        if rng.random() < 0.5 and pinned:  # completions
            for _ in range(int(rng.integers(1, len(pinned) + 1))):
                leaf, oleaf, _ = pinned.pop(int(rng.integers(0, len(pinned))))
                dev.release_path(leaf)
                ora.release_path(oleaf)
        if rng.random() < 0.3:
            k = int(rng.integers(0, 800))
            assert dev.evict(k) == ora.evict(k)
        v0 = len(dev.victim_log())
        src = torch.from_numpy(np.concatenate(batch_src) if batch_src else np.zeros((0, BPT), np.uint8)).cuda()
        vb = dev.stats()["victims"]
        new, freed = kv.sync(src if len(src) else None)
        st = kv.stats()
        assert st["rows"] - st["free"] == dev.resident_tokens == ora.resident_tokens, step
        assert new == sum(len(b) for b in batch_src)
        # every pinned request's rows: distinct per resident token and f(token, position)
        if pinned:
            slots = torch.tensor([lf.slot for lf, _, _ in pinned], dtype=torch.int32, device="cuda")
            ml = max(len(p) for _, _, p in pinned)
            table, lens, out = kv.gather(slots, len(pinned), ml, payload=True)
            out = out.cpu().numpy()
            for j, (_, _, p) in enumerate(pinned):
                assert int(lens[j]) == len(p)
                assert np.array_equal(out[j, :len(p)], _rows(p, np.arange(len(p)))), (step, j)
    assert dev.victim_log() == ora.victim_log()
    dev.close()


def test_wave_payload_counts_and_rows():
    """Fused waves at ~50K nodes with eviction every wave: rows in use track
    resident tokens, freed rows = the victims' tokens, a victim copy-out has
    the victims' payload, and every admitted request's table is complete."""
    import torch

    from paper_2605_08581_b200.kv import KvPool
    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig
    from paper_2605_08581_b200.wave import DevicePending, WaveEngine
    from traces import synth as S

    cap = 2_000_000
    eng = WaveEngine(CacheConfig(capacity_tokens=cap, policy=CachePolicy.DART, protect_budget=20),
                     SchedulerConfig(dispatch_budget=1024, cold_quota=16), S.C4.nseg, S.C4.sys_len, S.C4.chunk,
                     device=0)
    kv = KvPool(eng.t, cap + 2 * 1024 * S.C4.path_len, BPT)
    st = S.ShardStream("c4", 5, 1, 0)
    dev = torch.device("cuda", 0)
    prev = 0
    for w in range(12):
        eng.release(eng.leaf_slots, prev)
        pool = st.take(1024)
        nm, prev = eng.step(DevicePending.from_host(pool["ids"], pool["arrival"], pool["sk_off"], pool["sk"],
                                                    pool["reorderable"], pool["suffix"], dev))
        view = eng.cache_view()
        v0 = view.stats()["victims"]
        dst = torch.zeros((cap, BPT), dtype=torch.uint8, device=dev)
        new, freed = kv.sync(None, dst)
        s = kv.stats()
        assert s["rows"] - s["free"] == view.resident_tokens, w
        table, lens, _ = kv.gather(eng.leaf_slots, prev, S.C4.path_len)
        t = table.cpu().numpy()
        assert (lens.cpu().numpy() == S.C4.path_len).all()
        assert (t >= 0).all() and (t < kv.rows).all()
    assert s["freed"] > 100_000 and s["bytes_out"] == s["freed"] * BPT
    eng.close()
