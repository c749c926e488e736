"""The reference's toy Adam trainer on the GPU.

Mirrors ucp/models.py:101-366 (TrainerConfig, train_steps, first_diff,
states_equal): synthetic gradients from the integer-hash generator (stream
``grad.<step>`` of the tied leader's name) and a bias-corrected Adam update
in f64 with a fixed elementwise operation order, rounded to f32 after every
step. ``ucp_adam_step`` reproduces numpy's f64 arithmetic bit for bit
(explicit _rn intrinsics, no FMA contraction), so GPU training is
interchangeable with the reference's and resume equivalence (SPEC acceptance
2: train -> save -> reshard -> resume == train straight through) can be
checked at LLaMA scale.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._errors import ModelConfigError, from_status
from .engine import require_device, stream_ptr
from .spec import STATE_KINDS, DType, Tensor
from .synth import stream_base


@dataclass(frozen=True)
class TrainerConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    grad_seed: int = 2024
    steps: int = 100

    def validate(self) -> None:
        if not (0.0 < self.beta1 < 1.0 and 0.0 < self.beta2 < 1.0):
            raise ModelConfigError("betas must lie in (0, 1)")
        if self.lr <= 0 or self.eps <= 0:
            raise ModelConfigError("lr and eps must be positive")
        if self.steps < 0:
            raise ModelConfigError("steps must be >= 0")


def _pow_seq(base: float, n: int) -> float:
    out = 1.0
    for _ in range(n):
        out *= base
    return out


def adam_steps_device(w: torch.Tensor, m: torch.Tensor, v: torch.Tensor, name: str,
                      cfg: TrainerConfig, from_step: int, n: int, start: int = 0,
                      stream=None) -> None:
    """n in-place Adam steps on device f32 tensors holding flat elements
    [start, start + numel) of parameter ``name`` (its tied leader's name)."""
    lib = _native.lib()
    count = w.numel()
    for t in range(from_step, from_step + n):
        base = stream_base(cfg.grad_seed, name, f"grad.{t}")
        bc1 = 1.0 - _pow_seq(cfg.beta1, t + 1)
        bc2 = 1.0 - _pow_seq(cfg.beta2, t + 1)
        rc = lib.ucp_adam_step(ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(m.data_ptr()),
                               ctypes.c_void_p(v.data_ptr()), count, base, start, cfg.beta1,
                               1.0 - cfg.beta1, cfg.beta2, 1.0 - cfg.beta2, bc1, bc2, cfg.lr,
                               cfg.eps, stream_ptr(stream))
        if rc:
            raise from_status(rc, "ucp_adam_step")


def train_steps(state, cfg: TrainerConfig, from_step: int, n: int, *, device=None):
    """Advance a consolidated ModelState n steps on the GPU
    (ucp/models.py:296-328). Returns a new state; the input is untouched."""
    from .api import ModelState, ParamState

    cfg.validate()
    if state.step != from_step:
        raise ModelConfigError(f"state is at step {state.step}, expected from_step {from_step}")
    dev = require_device(device)
    spec = state.spec
    out: dict = {}
    for p in spec.params:
        lead = spec.tied_leader(p.name)
        if lead != p.name:
            out[p.name] = out[lead]
            continue
        ps = state.params[p.name]
        dev_t = [torch.from_numpy(np.ascontiguousarray(getattr(ps, k).data, dtype=np.float32)
                                  .reshape(-1)).to(dev) for k in STATE_KINDS]
        adam_steps_device(*dev_t, lead, cfg, from_step, n)
        host = [t.cpu().numpy().reshape(p.shape) for t in dev_t]
        out[p.name] = ParamState(*(Tensor(DType.F32, tuple(p.shape), h) for h in host))
    meta = dict(state.metadata)
    meta["iteration"] = from_step + n
    return ModelState(spec, out, from_step + n, meta)


def first_diff(a, b):
    """First differing element of two states, or None (ucp/models.py:338-362)."""
    if a.step != b.step:
        return ("<step>", "", -1, a.step, b.step)
    if set(a.params) != set(b.params):
        name = sorted(set(a.params) ^ set(b.params))[0]
        return (name, "", -1, name in a.params, name in b.params)
    for p in a.spec.params:
        for kind in STATE_KINDS:
            ta, tb = getattr(a.params[p.name], kind), getattr(b.params[p.name], kind)
            if tuple(ta.shape) != tuple(tb.shape) or ta.dtype is not tb.dtype:
                return (p.name, kind, -1, str(ta.shape), str(tb.shape))
            view = np.uint32 if ta.dtype is DType.F32 else np.uint16
            ba, bb = ta.data.reshape(-1).view(view), tb.data.reshape(-1).view(view)
            bad = np.flatnonzero(ba != bb)
            if bad.size:
                i = int(bad[0])
                return (p.name, kind, i, int(ba[i]), int(bb[i]))
    return None


def states_equal(a, b) -> bool:
    return first_diff(a, b) is None
