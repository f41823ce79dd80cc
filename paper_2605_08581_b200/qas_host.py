"""Host-side marshalling for one QAS round (no device code).

``marshal_round`` turns the reference's ``schedule_round(pending, active_set,
...)`` arguments (scheduler.py:192-197) into flat arrays: a CSR of skeletons
with segment ids remapped to a dense, order-preserving range ``[0, nseg)``
(so every ``(-pri, seg)`` tie-break of scheduler.py:124/141 is unchanged),
plus arrival times, ids and reorderable flags.  ``build_batch`` turns the
flat round outputs back into the reference's ``DispatchBatch``
(scheduler.py:69-80) holding the caller's own ``Request`` objects.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from .types import DispatchBatch, DispatchHint, SegmentCounters, export_anchor_offsets


@dataclass
class MarshaledRound:
    pending: list
    segs: np.ndarray  # dense id -> original segment id (sorted ascending)
    ids: np.ndarray  # int64 [P]
    arrival: np.ndarray  # float64 [P]
    sk_off: np.ndarray  # int64 [P+1]
    sk: np.ndarray  # int32 dense ids
    reorderable: np.ndarray  # uint8 [P]
    act_off: np.ndarray  # int64 [A+1]
    act_sk: np.ndarray  # int32 dense ids

    @property
    def nseg(self) -> int:
        return int(self.segs.shape[0])


def _csr(reqs: Sequence) -> tuple[np.ndarray, np.ndarray]:
    lens = np.fromiter((len(r.skeleton) for r in reqs), dtype=np.int64, count=len(reqs))
    off = np.zeros(len(reqs) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    flat = np.fromiter(
        (s for r in reqs for s in r.skeleton), dtype=np.int64, count=int(off[-1])
    )
    return off, flat


def marshal_round(pending: Sequence, active_set: Iterable) -> MarshaledRound:
    pending = list(pending)
    active = list(active_set)
    p_off, p_flat = _csr(pending)
    a_off, a_flat = _csr(active)
    segs = np.unique(np.concatenate([p_flat, a_flat]))
    sk = np.searchsorted(segs, p_flat).astype(np.int32)
    act_sk = np.searchsorted(segs, a_flat).astype(np.int32)
    ids = np.fromiter((r.id for r in pending), dtype=np.int64, count=len(pending))
    arrival = np.fromiter((r.arrival_time for r in pending), dtype=np.float64, count=len(pending))
    reo = np.fromiter((1 if r.reorderable else 0 for r in pending), dtype=np.uint8, count=len(pending))
    return MarshaledRound(pending, segs, ids, arrival, p_off, sk, reo, a_off, act_sk)


@dataclass
class RoundOutputs:
    """Flat outputs of one round, indices into the marshaled pending list."""

    hot: np.ndarray
    cold: np.ndarray
    aligned: np.ndarray  # dense ids, same CSR layout as sk
    sig: np.ndarray  # [P, kappa] dense ids
    siglen: np.ndarray  # [P]
    rank: np.ndarray  # [P]
    bucket: np.ndarray  # [P] bucket creation index
    bscore: np.ndarray  # [nbuckets] in creation order
    g: np.ndarray
    a: np.ndarray
    nd: np.ndarray
    prio: np.ndarray
    dom: np.ndarray


def build_batch(m: MarshaledRound, o: RoundOutputs) -> DispatchBatch:
    segs = m.segs.tolist()
    pending = m.pending
    hot = [pending[i] for i in o.hot.tolist()]
    cold = [pending[i] for i in o.cold.tolist()]
    g = o.g.tolist()
    a = o.a.tolist()
    nd = o.nd.tolist()
    gd = {segs[r]: c for r, c in enumerate(g) if c > 0}
    ad = {segs[r]: c for r, c in enumerate(a) if c > 0}
    nd_d = {segs[r]: c for r, c in enumerate(nd) if c > 0}
    prio = o.prio.tolist()
    priorities = {segs[r]: prio[r] for r in np.flatnonzero(o.dom).tolist()}
    siglen = o.siglen.tolist()
    sig_rows = o.sig.tolist()

    def sig_of(i: int) -> tuple[int, ...]:
        return tuple(segs[s] for s in sig_rows[i][: siglen[i]])

    # bucket_scores keyed by signature, in bucket creation order
    first_of_bucket: dict[int, int] = {}
    for i, b in enumerate(o.bucket.tolist()):
        if b not in first_of_bucket:
            first_of_bucket[b] = i
    bscore = o.bscore.tolist()
    scores = {sig_of(first_of_bucket[b]): bscore[b] for b in range(len(bscore))}

    hints: dict[int, DispatchHint] = {}
    sk_off = m.sk_off.tolist()
    aligned = o.aligned.tolist()
    rank = o.rank.tolist()
    for i in o.hot.tolist() + o.cold.tolist():
        req = pending[i]
        snapshot = {
            r: (gd.get(r, 0), ad.get(r, 0), nd_d.get(r, 0)) for r in set(req.skeleton)
        }
        hints[req.id] = DispatchHint(
            signature=sig_of(i),
            rank=rank[i],
            counter_snapshot=snapshot,
            anchor_offsets=export_anchor_offsets(req),
            aligned_skeleton=[segs[s] for s in aligned[sk_off[i] : sk_off[i + 1]]],
        )
    return DispatchBatch(
        hot=hot,
        cold=cold,
        hints=hints,
        priorities=priorities,
        counters=SegmentCounters(g=gd, a=ad, n=nd_d),
        bucket_scores=scores,
    )
