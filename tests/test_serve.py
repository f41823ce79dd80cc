"""The device serving loop (csrc/serve.cu, engine.py:141-266) and the native
trace reader (csrc/trace_io.cu, workload.py:258-313).

CPU: the native JSON-lines reader against the reference's load_trace
(restated verbatim in traces/refgen.py) on the golden traces, a generated
trace and every TraceFormatError case.
GPU: the whole serving loop on the device against the reference's recorded
engine runs (hits, admission order, every victim, TTFT)
and against the oracle-backed serving loop on generated traces (QPS sweep of
the 13B budget, eviction stress, decode attenuation, all policies).
"""

from __future__ import annotations

import io
import os

import numpy as np
import pytest

import golden_util as G
from traces.refgen import SegmentCatalog, WorkloadConfig, generate_trace, load_trace, save_trace


def _load_native(text: str, tmp_path, threads=0):
    from paper_2605_08581_b200.serve import TraceCSR

    p = tmp_path / "t.jsonl"
    p.write_text(text)
    return TraceCSR.load_jsonl(str(p), threads=threads)


def _assert_same(csr, tr):
    assert csr.n == len(tr.requests)
    assert csr.ids.tolist() == [r.id for r in tr.requests]
    assert csr.arrival.tolist() == [r.arrival_time for r in tr.requests]  # bit-exact floats
    assert [csr.sk[csr.sk_off[i]:csr.sk_off[i + 1]].tolist() for i in range(csr.n)] == [r.skeleton for r in tr.requests]
    assert csr.suffix.tolist() == [r.suffix_len for r in tr.requests]
    assert csr.reorderable.astype(bool).tolist() == [r.reorderable for r in tr.requests]
    assert csr.num_segments == tr.catalog.num_segments and csr.chunk_tokens == tr.catalog.chunk_tokens
    assert csr.sys_prefix_tokens == tr.catalog.sys_prefix_tokens and csr.hot_set == tuple(tr.catalog.hot_set)


@pytest.mark.parametrize("name", ["q40_s1", "q20_s1", "q10_s2"])
def test_native_reader_golden_traces(name, tmp_path):
    text = G.load("engine_runs.json.gz")["traces"][name]
    for threads in (1, 3, 0):
        _assert_same(_load_native(text, tmp_path, threads), load_trace(io.StringIO(text)))


def test_native_reader_generated(tmp_path):
    cat = SegmentCatalog(num_segments=5000, chunk_tokens=16, hot_set=tuple(range(0, 100, 3)), sys_prefix_tokens=7)
    tr = generate_trace(WorkloadConfig(qps=37.3, num_requests=20000, k=6, r_hot=0.6, zipf_alpha=1.1,
                                       suffix_tokens=13, reorderable=False, seed=4), cat)
    buf = io.StringIO()
    save_trace(tr, buf)
    text = buf.getvalue()
    csr = _load_native(text, tmp_path, threads=8)
    _assert_same(csr, load_trace(io.StringIO(text)))


def _reference_workload():
    """The reference's own workload module (its load_trace carries the line
    numbers): from /root/reference in the build container, or baseline/_ref."""
    import importlib
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for cand in ("/root/reference/pkg/src", os.path.join(root, "baseline", "_ref")):
        if os.path.isdir(os.path.join(cand, "prefixsim")):
            sys.path.insert(0, cand)
            try:
                return importlib.import_module("prefixsim.workload")
            finally:
                sys.path.remove(cand)
    pytest.skip("reference package not available")


HEADER = '{"catalog": {"num_segments": 10, "chunk_tokens": 4, "hot_set": [1], "sys_prefix_tokens": 2}}\n'


def _rec(i, t, sk, sfx=3, reo="true"):
    return f'{{"id": {i}, "arrival_time": {t}, "skeleton": {sk}, "suffix_tokens": {sfx}, "reorderable": {reo}}}\n'


@pytest.mark.parametrize("text,line", [
    ("", None),                                                            # empty file
    ('{"x": 1}\n' + _rec(0, 0.0, [1]), 1),                                 # missing catalog header
    (HEADER + _rec(0, 0.0, [1]) + '{"id": 1, "arrival_time": 0.1}\n', 3),  # bad request record
    (HEADER + _rec(0, 0.0, [1]) + _rec(0, 0.1, [2]), 3),                   # duplicate id
    (HEADER + _rec(0, 0.5, [1]) + _rec(1, 0.1, [2]), 3),                   # arrival decreases
    (HEADER + _rec(0, 0.0, [1]) + _rec(1, 0.1, [10]), 3),                  # unknown segment
    (HEADER + _rec(0, 0.0, [1]) + _rec(1, 0.1, [-1]) + _rec(1, 0.2, [2]), 3),  # the first offending line wins
    (HEADER + "\n" + _rec(0, 0.0, [1]) + "   \n" + _rec(2, 0.5, [3]) + _rec(2, 0.6, [4]), 6),  # blank lines counted
])
def test_native_reader_errors(text, line, tmp_path):
    from paper_2605_08581_b200.types import TraceFormatError as Mine

    W = _reference_workload()
    with pytest.raises(W.TraceFormatError) as ref:
        W.load_trace(io.StringIO(text))
    with pytest.raises(Mine) as mine:
        _load_native(text, tmp_path)
    if line is not None:
        assert str(ref.value).startswith(f"line {line}:")
        assert str(mine.value).startswith(f"line {line}:"), str(mine.value)
    assert isinstance(mine.value, ValueError)


def test_native_reader_good_edge_cases(tmp_path):
    text = HEADER + _rec(5, 0, [], sfx=0) + _rec(3, 0, [9, 9, 0], reo="false") + _rec(7, 1e-7, [2]) + "\n"
    _assert_same(_load_native(text, tmp_path), load_trace(io.StringIO(text)))


# ---------------------------------------------------------------- GPU: the serving loop


def _device_loop(trace, cfg):
    from paper_2605_08581_b200.serve import DeviceServingLoop, TraceCSR

    loop = DeviceServingLoop(cfg, TraceCSR.from_trace(trace))
    assert loop.run()
    return loop, loop.result()


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(G.load("engine_runs.json.gz")["runs"])))
def test_serving_loop_matches_reference_runs(case):
    """The reference's recorded run_simulation (Appendix A: C1 all policies,
    the 13B budget C2, the 10% eviction-stress capacity) replayed entirely by
    the device serving loop: hits, admission order, every victim, TTFTs."""
    run, trace, cfg = G.engine_case(case)
    loop, res = _device_loop(trace, cfg)
    assert res.trace.ids.tolist() == [r.id for r in trace.requests]
    obs = {
        "hit_rate": res.summary()["hit_rate"],
        "hits": res.hit_tokens.tolist(),
        "admission": res.admission(),
        "victims": loop.cache_view().victim_log(),
        "ttft": res.ttft.tolist(),
    }
    G.assert_engine_parity(obs, run)
    assert obs["ttft"] == run["ttft"]  # bit-identical, not just within 1e-6
    loop.close()


def _oracle_loop(trace, cfg):
    from oracle.oracle import OracleRadixCache, oracle_schedule_round
    from sim_harness import run_simulation

    holder = {}
    res = run_simulation(trace, cfg, cache_factory=OracleRadixCache, schedule_fn=oracle_schedule_round,
                         cache_hook=lambda c: holder.setdefault("c", c))
    return res, holder["c"]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [
    dict(qps=10.0), dict(qps=15.0), dict(qps=20.0), dict(qps=25.0), dict(qps=30.0),  # C2: 13B budget sweep
    dict(qps=60.0, cap=12557),                                # C5-like eviction stress, deep queue
    dict(qps=40.0, attenuate=True),                           # decode attenuation of the prefill rate
    dict(qps=40.0, policy="LRU_ACTIVE", cap=9000),
    dict(qps=40.0, policy="LFU", cap=9000),
    dict(qps=40.0, policy="LRU", cap=9000, budget=32, cold=4),
    dict(qps=200.0, cap=20000, budget=64, cold=8, n=3000),    # big waves, many in flight
])
def test_serving_loop_matches_oracle_loop(variant):
    from sim_harness import SimConfig
    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig

    cat = SegmentCatalog(num_segments=981, chunk_tokens=128, hot_set=tuple(range(20)), sys_prefix_tokens=28)
    tr = generate_trace(WorkloadConfig(qps=variant["qps"], num_requests=variant.get("n", 1200), k=5, r_hot=0.7,
                                       zipf_alpha=1.2, suffix_tokens=100, seed=int(variant["qps"]) + 1), cat)
    cfg = SimConfig(prefill_rate=1e4, decode_rate=4e4, output_tokens=32,
                    decode_attenuation_enabled=variant.get("attenuate", False),
                    cache=CacheConfig(capacity_tokens=variant.get("cap", 5760),
                                      policy=CachePolicy(variant.get("policy", "DART")), protect_budget=20),
                    scheduler=SchedulerConfig(window_s=0.05, dispatch_budget=variant.get("budget", 8),
                                              cold_quota=variant.get("cold", 2)))
    loop, res = _device_loop(tr, cfg)
    ref, cache = _oracle_loop(tr, cfg)
    assert res.hit_tokens.tolist() == [m.hit_tokens for m in ref.requests]
    assert res.admission() == [w.members for w in ref.waves]
    assert res.first_token.tolist() == [m.first_token for m in ref.requests]
    assert res.completion.tolist() == [m.completion for m in ref.requests]
    assert res.admit.tolist() == [m.admit for m in ref.requests]
    assert res.wave_duration.tolist() == [w.duration for w in ref.waves]
    assert loop.cache_view().victim_log() == cache.victim_log()
    s = res.summary()
    assert s["hit_rate"] == ref.run.hit_rate and s["p99"] == ref.run.p99 and s["makespan"] == ref.run.makespan
    assert s["reuse_hit_rate"] == ref.run.reuse_hit_rate and s["mean_wave_size"] == ref.run.mean_wave_size
    loop.close()


@pytest.mark.gpu
def test_serving_loop_from_jsonl_and_in_steps(tmp_path):
    """Native ingestion -> device loop, advanced a few waves at a time, equals
    the one-call run from the Python trace."""
    from paper_2605_08581_b200.serve import DeviceServingLoop, TraceCSR, run_simulation
    from sim_harness import SimConfig
    from paper_2605_08581_b200.types import CacheConfig, SchedulerConfig

    cat = SegmentCatalog(num_segments=300, chunk_tokens=32, hot_set=tuple(range(10)), sys_prefix_tokens=64)
    tr = generate_trace(WorkloadConfig(qps=80.0, num_requests=1500, k=8, r_hot=0.8, zipf_alpha=1.1,
                                       suffix_tokens=16, reorderable=False, seed=9), cat)
    p = tmp_path / "t.jsonl"
    with open(p, "w") as fh:
        save_trace(tr, fh)
    cfg = SimConfig(prefill_rate=2e4, decode_rate=4e4,
                    cache=CacheConfig(capacity_tokens=9000, protect_budget=8),
                    scheduler=SchedulerConfig(window_s=0.02, dispatch_budget=16, cold_quota=2))
    one = run_simulation(tr, cfg)
    loop = DeviceServingLoop(cfg, TraceCSR.load_jsonl(str(p)))
    steps = 0
    while not loop.run(max_waves=7):
        steps += 1
    two = loop.result()
    assert steps > 3
    for f in ("admit", "first_token", "completion", "hit_tokens", "wave_members", "wave_off", "wave_duration"):
        assert np.array_equal(getattr(one, f), getattr(two, f)), f
    loop.close()


@pytest.mark.gpu
def test_serving_loop_errors():
    from paper_2605_08581_b200.serve import run_simulation
    from sim_harness import SimConfig
    from paper_2605_08581_b200.types import CacheConfig, SchedulerConfig, SimulationError

    cat = SegmentCatalog(num_segments=50, chunk_tokens=128, hot_set=(0,), sys_prefix_tokens=28)
    tr = generate_trace(WorkloadConfig(qps=10.0, num_requests=10, k=5, r_hot=0.5, zipf_alpha=1.2), cat)
    cfg = SimConfig(prefill_rate=1e4, decode_rate=4e4, cache=CacheConfig(capacity_tokens=500),
                    scheduler=SchedulerConfig())
    with pytest.raises(SimulationError, match="exceeds cache capacity"):
        run_simulation(tr, cfg)


@pytest.mark.parametrize("variant", [dict(qps=20.0, cap=5760), dict(qps=60.0, cap=12557, attenuate=True),
                                     dict(qps=40.0, cap=9000, policy="LRU_ACTIVE")])
def test_oracle_serve_loop_matches_harness(variant):
    """oracle/serve_loop.py (the array-based checker used at scale) against the
    per-request restatement of engine.py in tests/sim_harness.py (CPU)."""
    from oracle.serve_loop import oracle_serve
    from paper_2605_08581_b200.serve import TraceCSR
    from paper_2605_08581_b200.types import CacheConfig, CachePolicy, SchedulerConfig
    from sim_harness import SimConfig

    cat = SegmentCatalog(num_segments=981, chunk_tokens=128, hot_set=tuple(range(20)), sys_prefix_tokens=28)
    tr = generate_trace(WorkloadConfig(qps=variant["qps"], num_requests=800, k=5, r_hot=0.7, zipf_alpha=1.2,
                                       suffix_tokens=100, seed=3), cat)
    cfg = SimConfig(prefill_rate=1e4, decode_rate=4e4, decode_attenuation_enabled=variant.get("attenuate", False),
                    cache=CacheConfig(capacity_tokens=variant["cap"], policy=CachePolicy(variant.get("policy", "DART")),
                                      protect_budget=20),
                    scheduler=SchedulerConfig(window_s=0.05, dispatch_budget=8, cold_quota=2))
    o = oracle_serve(TraceCSR.from_trace(tr), cfg)
    ref, cache = _oracle_loop(tr, cfg)
    assert o["hit"].tolist() == [m.hit_tokens for m in ref.requests]
    assert o["first_token"].tolist() == [m.first_token for m in ref.requests]
    assert o["completion"].tolist() == [m.completion for m in ref.requests]
    ids = TraceCSR.from_trace(tr).ids
    sizes = np.cumsum(np.concatenate([[0], o["wave_sizes"]]))
    assert [ids[o["wave_members"][sizes[w]:sizes[w + 1]]].tolist() for w in range(len(sizes) - 1)] == \
        [w.members for w in ref.waves]
    assert o["victims"].tolist() == cache.victim_log()
