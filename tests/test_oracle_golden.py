"""Pin the CPU oracle (oracle/) to the reference via tests/golden/ (CPU only).

The fixtures were produced by the reference itself (tools/make_golden.py);
these tests prove the C restatement reproduces them bit for bit before it is
trusted as the checker for the device path.
"""

from __future__ import annotations

import pytest

import golden_util as G
from oracle.oracle import OracleRadixCache, oracle_schedule_round


@pytest.mark.parametrize("case", range(len(G.load("dart_ops.json.gz"))))
def test_oracle_dart_ops(case):
    G.replay_dart_case(G.load("dart_ops.json.gz")[case], OracleRadixCache)


def test_oracle_qas_rounds():
    for i, case in enumerate(G.load("qas_rounds.json.gz")):
        pending, active, cfg = G.qas_case(case)
        batch = oracle_schedule_round(pending, active, cfg, 0.0)
        try:
            G.assert_qas_case(case, batch)
        except AssertionError as e:  # pragma: no cover - diagnostic
            raise AssertionError(f"round {i}: {e}") from e


@pytest.mark.parametrize("case", range(len(G.load("engine_runs.json.gz")["runs"])))
def test_oracle_engine_runs(case):
    obs, run = G.run_engine_case(case, OracleRadixCache, oracle_schedule_round)
    G.assert_engine_parity(obs, run)
