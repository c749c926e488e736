"""Bind this package into an imported reference ``ucp`` package in place.

The reference binds ``convert``/``load``/``resume``/``union``/``ucp_info`` at
import time in several modules (SURVEY §8b "How to hot-swap"), so a user who
wants the GPU path under unchanged reference code patches every binding site:

    import ucp, paper_2406_18820_b200.hotswap as hs
    undo = hs.install(ucp)       # ucp.convert & co. now run on the B200
    ...
    undo()

The adapters translate at the boundary only, without copying payloads:
- arguments: the reference's ``DType`` becomes ours by name; its
  ``ParallelConfig``/``ParamSpec``/``RecordMeta``/``FragmentMsg`` objects are
  read by duck typing (``layout.kind_of``/``zero_of``);
- results: ``LoadedWorld``/``WorldShard``/``LoadStats``/``Tensor``/
  ``RecordMeta``/``AtomicCheckpoint``/``UcpInfo``/``ModelSpec`` are rebuilt
  as the reference's own classes around the same numpy buffers, so identity
  checks such as ``t.dtype is DType.F32`` (ucp/oracle.py:219) and dataclass
  equality against ``enumerate_rank_records`` (pkg/tests/test_load.py:105-112)
  hold;
- errors: each of our exceptions is re-raised as the reference class of the
  same name (ucp/errors.py), chained to the original.

``ucp.parallel.extract_fragment`` and ``ucp.oracle`` are deliberately left
alone: the reference's tests use them as the expected value and the
partitioner uses them to generate inputs.
"""

from __future__ import annotations

import dataclasses
import functools
import sys

from . import api
from ._errors import UcpError
from .spec import DType, spec_to_dict

# (module path relative to the reference package, names bound there);
# ucp/__init__.py:10-18,37, ucp/convert.py, ucp/load.py:23-31,
# ucp/verify.py:29-30, ucp/bench.py:22-23, ucp/cli.py:18-20
SITES = (
    ("", ("convert", "union", "load", "resume", "ucp_info", "conversions_invoked")),
    ("convert", ("convert", "union", "conversions_invoked")),
    ("load", ("load", "resume", "extract_fragment", "ucp_info")),
    ("verify", ("convert", "load", "resume")),
    ("bench", ("convert", "load")),
    ("cli", ("convert", "load", "resume")),
)


class _Adapter:
    """Type translation between this package and one reference package."""

    def __init__(self, ucp):
        self.ucp = ucp
        self.m = {name: sys.modules[f"{ucp.__name__}.{name}"]
                  for name in ("convert", "load", "tensor", "parallel", "models", "errors")}

    # -- arguments
    @staticmethod
    def dtype_in(dt) -> DType:
        return DType[dt.name]

    # -- results
    def spec_out(self, spec):
        return self.m["models"].spec_from_dict(spec_to_dict(spec))

    def meta_out(self, meta):
        RM = self.m["parallel"].RecordMeta
        return RM(**{f.name: getattr(meta, f.name) for f in dataclasses.fields(RM)})

    def tensor_out(self, t):
        T, D = self.m["tensor"].Tensor, self.m["tensor"].DType
        return T(D[t.dtype.name], tuple(t.shape), t.data)

    def stats_out(self, st):
        LS = self.m["load"].LoadStats
        return LS(**{f.name: getattr(st, f.name) for f in dataclasses.fields(LS)})

    def world_out(self, w, cfg):
        L = self.m["load"]
        shards = {g: [L.WorldShard(self.meta_out(s.meta), self.tensor_out(s.tensor)) for s in v]
                  for g, v in w.shards.items()}
        return L.LoadedWorld(cfg, self.spec_out(w.spec), w.step, dict(w.metadata), shards,
                             self.stats_out(w.stats))

    def atomic_out(self, a):
        return self.m["convert"].AtomicCheckpoint(a.root, self.spec_out(a.spec), a.step,
                                                  dict(a.metadata), a.source_fingerprint)

    def info_out(self, info, cfg):
        return self.m["load"].UcpInfo(
            cfg, {g: [self.meta_out(m) for m in v] for g, v in info.records.items()})

    def error_out(self, e: UcpError) -> Exception:
        cls = getattr(self.m["errors"], type(e).__name__, self.m["errors"].UcpError)
        return cls(str(e))


def _guard(ad: _Adapter, fn):
    @functools.wraps(fn)
    def wrapped(*a, **k):
        try:
            return fn(*a, **k)
        except UcpError as e:
            raise ad.error_out(e) from e
    return wrapped


def adapters(ucp) -> dict:
    """The reference-typed wrappers, by reference name."""
    ad = _Adapter(ucp)

    def convert(src, out_dir, n_workers=1, inner=1, strict_replicate=True):
        return ad.atomic_out(api.convert(src, out_dir, n_workers, inner, strict_replicate))

    def load(atomic_root, tgt, dtype=None, bypass=True):
        dt = DType.F32 if dtype is None else ad.dtype_in(dtype)
        return ad.world_out(api.load(atomic_root, tgt, dt, bypass), tgt)

    def resume(src_root, tgt, scratch, n_workers=1, inner=1, dtype=None, bypass=True):
        dt = DType.F32 if dtype is None else ad.dtype_in(dtype)
        return ad.world_out(api.resume(src_root, tgt, scratch, n_workers, inner, dt, bypass), tgt)

    def ucp_info(spec, cfg):
        return ad.info_out(api.ucp_info(spec, cfg), cfg)

    out = {"convert": convert, "load": load, "resume": resume, "ucp_info": ucp_info,
           "union": api.union, "extract_fragment": api.extract_fragment,
           "conversions_invoked": api.conversions_invoked}
    return {k: _guard(ad, v) for k, v in out.items()}


def install(ucp):
    """Patch every binding site of the reference package ``ucp`` (an imported
    module object); returns a callable restoring the originals."""
    fns = adapters(ucp)
    saved = []
    for sub, names in SITES:
        mod = ucp if not sub else sys.modules.get(f"{ucp.__name__}.{sub}")
        if mod is None:
            continue
        for n in names:
            if hasattr(mod, n):
                saved.append((mod, n, getattr(mod, n)))
                setattr(mod, n, fns[n])

    def uninstall():
        for mod, n, orig in reversed(saved):
            setattr(mod, n, orig)
    return uninstall
