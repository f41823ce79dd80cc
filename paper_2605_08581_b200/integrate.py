"""Drop-in injection into the reference's serving loop.

The reference resolves its cache and scheduler through module-level names
(engine.py:18-28, used at engine.py:157 and 189), so the drop-in is a module
attribute swap:

    import prefixsim
    from paper_2605_08581_b200.integrate import install
    install(prefixsim)              # RadixCache -> DeviceRadixCache, schedule_round -> device QAS
    prefixsim.engine.run_simulation(trace, config)   # unchanged reference loop

The device cache then raises the reference's own CapacityError /
ReleaseError classes (the engine catches prefixsim.kvcache.CapacityError,
engine.py:209), and accepts the reference's CacheConfig / Anchor / NodeKind
objects (they are read by value).  ``uninstall`` restores the originals.
"""

from __future__ import annotations

from . import dart as _dart

_SAVED: dict = {}


def install(prefixsim_pkg, cache: bool = True, scheduler: bool = True) -> None:
    engine = prefixsim_pkg.engine
    kv = prefixsim_pkg.kvcache
    _SAVED.setdefault("RadixCache", engine.RadixCache)
    _SAVED.setdefault("schedule_round", engine.schedule_round)
    _SAVED.setdefault("errors", dict(_dart.ERRORS))
    _dart.ERRORS["capacity"] = kv.CapacityError
    _dart.ERRORS["release"] = kv.ReleaseError
    if cache:
        engine.RadixCache = _dart.DeviceRadixCache
    if scheduler:
        from .qas import schedule_round

        engine.schedule_round = schedule_round


def uninstall(prefixsim_pkg) -> None:
    engine = prefixsim_pkg.engine
    if "RadixCache" in _SAVED:
        engine.RadixCache = _SAVED.pop("RadixCache")
    if "schedule_round" in _SAVED:
        engine.schedule_round = _SAVED.pop("schedule_round")
    if "errors" in _SAVED:
        _dart.ERRORS.update(_SAVED.pop("errors"))
