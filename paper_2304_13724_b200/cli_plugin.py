"""The B200 trainer as a variant of the reference CLI.

The reference's command line picks its trainer from a table,
``VARIANTS = {"bgmf": train_blocked, "cmf": ..., "cpmf": ...}``
(/root/reference/pkg/src/blockmf/cli.py:47-51), and calls
``VARIANTS[name](train, cfg, test, early_stop=..., timing=...)`` (cli.py:165-177;
``benchmark``, cli.py:217-219, calls ``VARIANTS[v](d, cfg)``).  ``register()``
adds ``"bgmf-b200"`` to that table -- the plug point SURVEY §8(f)-2 names -- so
``blockmf train --variant bgmf-b200`` (and anything else that looks variants
up there) trains on the GPU while the CLI's loading, splitting, trace / model
writers and reports stay the reference's own.

``train_variant`` takes the caller's objects as they come: this package's
``RatingsDataset`` / ``TrainConfig`` go straight to ``train_blocked``; the
reference package's own (the unmodified reference installed next to this one)
are converted field by field -- the dataset arrays, the config's dataclass
fields, the inner schedule by class name and fields -- and the result comes
back as the caller's ``TrainResult`` / ``FactorModel`` / ``ConvergenceTrace``
/ ``TraceStep`` classes, so the reference's writers (write_trace, save_model)
and reports accept it unchanged.
"""

from __future__ import annotations

import dataclasses
import importlib
import sys

from . import core as _core
from .trainer import train_blocked

VARIANT = "bgmf-b200"


def _schedule(s):
    """A schedule object of either package -> this package's equivalent."""
    if isinstance(s, _core.InnerSchedule):
        return s
    cls = getattr(_core, type(s).__name__, None)
    if cls is None or not dataclasses.is_dataclass(s):
        raise TypeError(f"unsupported inner schedule {s!r}")
    return cls(**{f.name: getattr(s, f.name) for f in dataclasses.fields(s)})


def to_config(cfg) -> _core.TrainConfig:
    if isinstance(cfg, _core.TrainConfig):
        return cfg
    kw = {f.name: getattr(cfg, f.name) for f in dataclasses.fields(_core.TrainConfig)
          if hasattr(cfg, f.name)}
    kw["inner_schedule"] = _schedule(kw.get("inner_schedule", _core.Constant(1)))
    return _core.TrainConfig(**kw)


def to_dataset(d) -> _core.RatingsDataset | None:
    if d is None or isinstance(d, _core.RatingsDataset):
        return d
    return _core.RatingsDataset(d.n, d.m, d.rows, d.cols, d.values)


def _caller_modules(d):
    """The caller's core and trainer modules (the package its dataset came from)."""
    pkg = type(d).__module__.rsplit(".", 1)[0]
    return importlib.import_module(pkg + ".core"), importlib.import_module(pkg + ".trainer")


def to_caller_result(res, d):
    """This package's TrainResult -> the classes of the package ``d`` came from."""
    if isinstance(d, _core.RatingsDataset):
        return res
    rcore, rtrainer = _caller_modules(d)
    trace = rcore.ConvergenceTrace()
    for s in res.trace:
        trace.append(rcore.TraceStep(**{f.name: getattr(s, f.name)
                                       for f in dataclasses.fields(rcore.TraceStep)}))
    model = rcore.FactorModel(res.model.u, res.model.v)
    return rtrainer.TrainResult(model=model, trace=trace, stop_reason=res.stop_reason)


def train_variant(d, cfg, test=None, *, early_stop: bool = True, timing: bool = True, **kw):
    """``VARIANTS["bgmf-b200"]``: the reference trainer signature
    (trainer.py:76-184), trained by this package's GPU engine."""
    res = train_blocked(to_dataset(d), to_config(cfg), to_dataset(test),
                        early_stop=early_stop, timing=timing, **kw)
    return to_caller_result(res, d)


def register(variants: dict | None = None) -> dict:
    """Add ``"bgmf-b200"`` to a CLI variant table (default: ``blockmf.cli.VARIANTS``
    of the importable ``blockmf``).  Call before the CLI builds its parser
    (its ``--variant`` choices are read from the table)."""
    if variants is None:
        variants = (sys.modules.get("blockmf.cli") or importlib.import_module("blockmf.cli")).VARIANTS
    variants[VARIANT] = train_variant
    return variants
