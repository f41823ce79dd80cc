"""The benchmark workloads (traces/synth.py) and the replica routing of one
global stream: CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from traces import synth as S


def test_c3_shape_and_chains():
    rng = np.random.default_rng(3)
    p = S.make_pool("c3", 100, 5000, rng)
    sk = p["sk"].reshape(-1, 40).astype(np.int64)
    assert p["ids"][0] == 100 and len(p["ids"]) == 5000
    assert np.all(p["reorderable"] == 0) and np.all(p["suffix"] == 128)
    assert sk.min() >= 0 and sk.max() < (1 << 20)
    assert all(len(set(r)) == 40 for r in sk.tolist())  # distinct within a request
    assert sk[:, 0].max() < 1024  # slot 0 over the hot set
    # slot d < 24 is a child of slot d-1 (one of its 8 hash children)
    kids = S.splitmix64(8 * sk[:, :23, None].astype(np.uint64) + np.arange(8, dtype=np.uint64)) % np.uint64(1 << 20)
    is_child = (kids.astype(np.int64) == sk[:, 1:24, None]).any(axis=2)
    assert is_child.mean() > 0.999
    # Zipf-skewed: the most popular root carries far more than 1/1024 of requests
    assert np.bincount(sk[:, 0]).max() / len(sk) > 0.1
    # deep sharing at the top, unique tails at the bottom
    assert len({tuple(r) for r in sk[:, :2].tolist()}) < 0.5 * len(sk)
    assert len({tuple(r) for r in sk[:, :12].tolist()}) > 0.95 * len(sk)


def test_generators_are_deterministic():
    for w in ("c3", "mu1m", "c4"):
        a = S.make_pool(w, 0, 777, np.random.default_rng(11))
        b = S.make_pool(w, 0, 777, np.random.default_rng(11))
        for k in a:
            assert np.array_equal(a[k], b[k])


def test_c4_hot_and_cold():
    p = S.make_pool("c4", 0, 20000, np.random.default_rng(5))
    sk = p["sk"].reshape(-1, 5)
    hot = sk[:, 0] < 1000
    assert 0.65 < hot.mean() < 0.75
    assert np.all(sk[~hot] >= 1000)  # cold requests avoid the hot set
    assert all(len(set(r)) == 5 for r in sk.tolist())


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shard_streams_partition_one_global_stream(world):
    n = 3000
    glob = S.make_pool("c3", 0, 1 << 15, np.random.default_rng(42))
    shards = []
    for r in range(world):
        st = S.ShardStream("c3", 42, world, r)
        got = st.take(n // world)
        shards.append(got)
        want = np.flatnonzero(S.route(glob, world) == r)[: n // world]
        assert np.array_equal(got["ids"], glob["ids"][want])  # the shard's requests, in stream order
        assert np.array_equal(got["sk"], S.select(glob, want)["sk"])
        if world > 1:
            assert np.all(S.route(got, world) == r)
    ids = np.concatenate([s["ids"] for s in shards])
    assert len(np.unique(ids)) == len(ids)


def test_take_is_sequential():
    st = S.ShardStream("mu1m", 1, 2, 1)
    a, b = st.take(100), st.take(100)
    st2 = S.ShardStream("mu1m", 1, 2, 1)
    c = st2.take(200)
    assert np.array_equal(np.concatenate([a["ids"], b["ids"]]), c["ids"])
    assert np.array_equal(np.concatenate([a["sk"], b["sk"]]), c["sk"])
