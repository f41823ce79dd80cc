"""The drop-in inside the UNMODIFIED reference serving loop.

Uses the reference package installed offline into baseline/_ref (git-ignored;
present on the GPU box when the driver ships it, skipped otherwise):
``install(prefixsim)`` swaps prefixsim.engine.RadixCache / schedule_round for
the device implementations, then the reference's own run_simulation replays
the SURVEY.md Appendix A configurations and must reproduce the reference's
recorded hits, admission order, victims and TTFTs bit for bit.
"""

from __future__ import annotations

import os
import sys

import pytest

import golden_util as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def prefixsim():
    if not os.path.isdir(os.path.join(REF, "prefixsim")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import prefixsim as P  # noqa: F401
        import prefixsim.engine  # noqa: F401
        import prefixsim.kvcache  # noqa: F401
    finally:
        sys.path.remove(REF)
    from paper_2605_08581_b200.integrate import install, uninstall

    install(P)
    yield P
    uninstall(P)


@pytest.mark.parametrize("case", range(len(G.load("engine_runs.json.gz")["runs"])))
def test_reference_engine_with_device_path(prefixsim, case):
    import hashlib
    import json

    from prefixsim.experiment import SimSpec, WorkloadSpec
    from prefixsim.kvcache import CachePolicy
    from prefixsim.workload import generate_trace

    run = G.load("engine_runs.json.gz")["runs"][case]
    victims: list[int] = []
    created: list = []
    DC = prefixsim.engine.RadixCache  # the device cache after install()

    class Recording(DC):
        def __init__(self, cfg):
            super().__init__(cfg)
            created.append(self)

    prefixsim.engine.RadixCache = Recording
    try:
        wl = WorkloadSpec()
        tr = generate_trace(wl.config(run["qps"], run["seed"]), wl.catalog())
        res = prefixsim.engine.run_simulation(
            tr, SimSpec(capacity_tokens=run["capacity"]).config(CachePolicy(run["policy"]), 2)
        )
    finally:
        prefixsim.engine.RadixCache = DC
    victims = created[0].victim_log()
    H = lambda x: hashlib.sha256(json.dumps(x).encode()).hexdigest()[:16]  # noqa: E731
    assert res.run.hit_rate == run["hit_rate"]
    assert [m.hit_tokens for m in res.requests] == run["hits"]
    assert [w.members for w in res.waves] == run["admission"]
    assert victims == run["victims"]
    assert H([m.ttft for m in res.requests]) == run["digest"][5]
