"""Device QAS: ``schedule_round`` (scheduler.py:192-273) on the B200.

Same signature and result as the reference: ``schedule_round(pending,
active_set, config, now) -> DispatchBatch`` holding the caller's own Request
objects.  The round itself (counters, front alignment, signatures, buckets,
scores, hot/cold lanes, dispatch priorities) runs as the device passes of
csrc/qas.cu; this module only marshals the request list.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from ._lib import check
from .qas_host import RoundOutputs, build_batch, marshal_round
from .types import DispatchBatch, SchedulerConfig


class _QasCfg(C.Structure):
    _fields_ = [
        ("dispatch_budget", C.c_int64),
        ("cold_quota", C.c_int64),
        ("front_width", C.c_int64),
        ("signature_size", C.c_int64),
        ("w_g", C.c_double),
        ("w_a", C.c_double),
        ("w_n", C.c_double),
        ("alpha_size", C.c_double),
        ("beta_util", C.c_double),
    ]


_WARNED = False


def warn_nonintegral(config: SchedulerConfig) -> None:
    """Non-integral weights (w_g, w_a, w_n): the device sums each bucket's
    utility terms in ascending segment order, the reference in Python ``set``
    iteration order (scheduler.py:163-169), so a score may differ in its last
    bit and, on an exact tie, the dispatch order with it.  Integral weights
    (the reference's defaults) are summed exactly in int64: identical."""
    global _WARNED
    w = config.weights
    if _WARNED or all(float(x).is_integer() for x in (w.w_g, w.w_a, w.w_n)):
        return
    import warnings

    warnings.warn("non-integral QAS weights: bucket utilities are summed in ascending segment order, the "
                  "reference in set order; scores may differ in the last bit", RuntimeWarning, stacklevel=3)
    _WARNED = True


def _cfg(config: SchedulerConfig) -> _QasCfg:
    warn_nonintegral(config)
    w = config.weights
    return _QasCfg(config.dispatch_budget, config.cold_quota, config.front_width, config.signature_size,
                   w.w_g, w.w_a, w.w_n, config.alpha_size, config.beta_util)


class DeviceScheduler:
    """Owns the device buffers of one QAS instance (one per GPU)."""

    def __init__(self, device: int = 0):
        _lib.require_device()
        self._L = _lib.lib()
        self._h = self._L.prism_qas_create(device)
        if not self._h:
            raise _lib.PrismError(_lib.last_error())

    def set_small(self, on: bool | int) -> None:
        """One-CTA rounds for small pending sets with integral weights.
        True: the default cutoff; False: never; an int: the largest P (<= 4096)."""
        self._L.prism_qas_set_small.argtypes = [C.c_void_p, C.c_int32]
        max_p = (1 if on else 0) if isinstance(on, bool) else int(on)
        check(self._L.prism_qas_set_small(self._h, max_p))

    _TUNE = {"max_p": 0, "grid": 1, "per_cta": 2}

    def tune(self, **kw) -> None:
        """One-launch round shape: max_p, grid (CTAs, 0 = auto), per_cta."""
        self._L.prism_qas_tune.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]
        for k, v in kw.items():
            check(self._L.prism_qas_tune(self._h, self._TUNE[k], int(v), None))

    def last_grid(self) -> int:
        """CTAs of the last one-launch round."""
        out = C.c_int64(0)
        self._L.prism_qas_tune.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]
        check(self._L.prism_qas_tune(self._h, 3, 0, C.addressof(out)))
        return int(out.value)

    def profile(self, on: bool) -> None:
        self._L.prism_qas_profile.argtypes = [C.c_void_p, C.c_int32]
        check(self._L.prism_qas_profile(self._h, 1 if on else 0))

    def small_timeline(self) -> list[int]:
        """ns from kernel start to the end of each one-CTA phase (last profiled round)."""
        out = np.zeros(11, np.int64)
        self._L.prism_qas_small_timeline.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        check(self._L.prism_qas_small_timeline(self._h, out.ctypes.data, 11))
        return [int(x) for x in out]

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.prism_qas_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover
            pass

    def round_arrays(self, m, config: SchedulerConfig) -> RoundOutputs:
        if config.cold_quota > config.dispatch_budget:
            raise ValueError("cold_quota must be <= dispatch_budget")
        P = len(m.pending)
        kappa = config.signature_size
        nseg = m.nseg
        n1 = max(P, 1)
        s1 = max(nseg, 1)
        hot = np.zeros(n1, np.int64)
        cold = np.zeros(n1, np.int64)
        nhot = np.zeros(1, np.int64)
        ncold = np.zeros(1, np.int64)
        aligned = np.zeros(max(len(m.sk), 1), np.int32)
        sig = np.zeros(n1 * kappa, np.int32)
        siglen = np.zeros(n1, np.int32)
        rank = np.zeros(n1, np.int64)
        bucket = np.zeros(n1, np.int64)
        bscore = np.zeros(n1, np.float64)
        nb = np.zeros(1, np.int64)
        g = np.zeros(s1, np.int32)
        a = np.zeros(s1, np.int32)
        nd = np.zeros(s1, np.int32)
        prio = np.zeros(s1, np.float64)
        dom = np.zeros(s1, np.uint8)
        sk = m.sk if len(m.sk) else np.zeros(1, np.int32)
        ask = m.act_sk if len(m.act_sk) else np.zeros(1, np.int32)
        ids = m.ids if P else np.zeros(1, np.int64)
        arr = m.arrival if P else np.zeros(1, np.float64)
        reo = m.reorderable if P else np.zeros(1, np.uint8)
        cfg = _cfg(config)
        p = lambda x: x.ctypes.data  # noqa: E731
        check(self._L.prism_qas_round(
            self._h, P, p(ids), p(arr), p(m.sk_off), p(sk), p(reo), len(m.act_off) - 1, p(m.act_off), p(ask),
            nseg, C.addressof(cfg), p(hot), p(nhot), p(cold), p(ncold), p(aligned), p(sig), p(siglen),
            p(rank), p(bucket), p(bscore), p(nb), p(g), p(a), p(nd), p(prio), p(dom),
        ))
        return RoundOutputs(
            hot=hot[: nhot[0]], cold=cold[: ncold[0]], aligned=aligned[: len(m.sk)],
            sig=sig[: P * kappa].reshape(P, kappa), siglen=siglen[:P], rank=rank[:P], bucket=bucket[:P],
            bscore=bscore[: nb[0]], g=g[:nseg], a=a[:nseg], nd=nd[:nseg], prio=prio[:nseg], dom=dom[:nseg],
        )

    def schedule_round(self, pending, active_set, config: SchedulerConfig, now: float = 0.0) -> DispatchBatch:
        m = marshal_round(pending, active_set)
        return build_batch(m, self.round_arrays(m, config))


_LOCAL = threading.local()


def _default() -> DeviceScheduler:
    s = getattr(_LOCAL, "sched", None)
    if s is None:
        s = DeviceScheduler()
        _LOCAL.sched = s
    return s


def schedule_round(pending, active_set, config: SchedulerConfig, now: float) -> DispatchBatch:
    """Drop-in for prefixsim.scheduler.schedule_round (scheduler.py:192-273)."""
    return _default().schedule_round(pending, active_set, config, now)
