"""Paths and skeletons beyond the shared-memory staging sizes.

The reference's match_prefix / insert_path have no length limit
(kvcache.py:146-241): paths longer than the 16,384 tokens the ordered commit
stages in shared memory are read from HBM in place; skeletons of ~100
segments take the block-wide QAS alignment and the ordered commit.  Compared
with the oracle op by op / wave by wave.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle.oracle import OracleRadixCache
from paper_2605_08581_b200.types import Anchor, CacheConfig, CachePolicy, CapacityError, NodeKind

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(2))
def test_100k_token_paths_per_call(seed):
    from paper_2605_08581_b200.dart import DeviceRadixCache

    rng = np.random.default_rng(seed)
    cfg = CacheConfig(capacity_tokens=400_000, policy=CachePolicy.DART, protect_budget=3)
    dev, ora = DeviceRadixCache(cfg), OracleRadixCache(cfg)
    base = [int(x) for x in rng.integers(0, 10**6, size=120_000)]
    pinned = []
    for step in range(24):
        L = int(rng.choice([17_000, 40_000, 100_000, 120_000]))
        cut = int(rng.integers(0, L))
        path = base[:cut] + [int(x) for x in rng.integers(10**6, 2 * 10**6, size=L - cut)]
        offs = sorted({int(x) for x in rng.integers(1, L, size=int(rng.integers(1, 100)))})
        anchors = [Anchor(o, NodeKind.REUSABLE, int(rng.integers(0, 50))) for o in offs]
        assert dev.match_prefix(path)[0] == ora.match_prefix(path)[0], step
        try:
            leaf = dev.insert_path(path, anchors)
        except CapacityError:
            with pytest.raises(CapacityError):
                ora.insert_path(path, anchors)
            continue
        oleaf = ora.insert_path(path, anchors)
        assert leaf.node_id == oleaf.node_id
        pinned.append((leaf, oleaf))
        if len(pinned) > 2:
            a, b = pinned.pop(0)
            dev.release_path(a)
            ora.release_path(b)
        if step % 5 == 4:
            pri = {int(s): float(rng.integers(1, 9)) for s in rng.integers(0, 50, size=10)}
            assert dev.set_protection(pri) == ora.set_protection(pri)
    assert dev.resident_tokens == ora.resident_tokens
    assert dev.victim_log() == ora.victim_log()
    assert dev.debug_nodes() == ora.debug_nodes()
    dev.close()


@pytest.mark.parametrize("mode", [0, 1])
def test_k100_skeletons_fused_wave(mode):
    from test_wave_fused import run_case

    run_case(4, CachePolicy.DART, mode=mode, nseg=5000, hot=8, kmin=90, kmax=110, suffixes=(0, 8), wave=12,
             nwaves=6, cap=9000, chunk=4)
