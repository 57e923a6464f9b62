"""MAE random patch masking (mirror of cropload/masking.py:21-65) on the GPU.

``sample_mask`` returns exactly the reference's sorted masked ids
(masking.py:48-56); the batched loader path also emits the MAE conventions
``ids_keep = sorted(complement(mask))`` and
``ids_restore = argsort(concat(ids_keep, mask))``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ConfigError
from .schedule import ScheduleScheme, params_for_epoch

_GAMMA = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


@dataclass(frozen=True)
class MaskSpec:
    grid: int
    ratio: float

    def __post_init__(self):
        if self.grid < 1:
            raise ConfigError(f"grid must be >= 1, got {self.grid}")
        if not 0.0 <= self.ratio <= 1.0:
            raise ConfigError(f"mask ratio out of [0, 1]: {self.ratio}")

    @classmethod
    def from_resolution(cls, resolution: int, patch: int, ratio: float) -> "MaskSpec":
        if patch < 1 or resolution % patch != 0:
            raise ConfigError(f"patch size {patch} does not divide resolution {resolution}")
        return cls(resolution // patch, ratio)

    @property
    def tokens(self) -> int:
        return self.grid * self.grid

    @property
    def masked_count(self) -> int:
        return int(math.floor(self.ratio * self.tokens + 0.5))


def sample_masks(states, spec: MaskSpec, device=None, want_ids=False):
    """Masks for a batch of DOMAIN_MASK stream states (uint64) on the GPU.
    Returns torch tensors (mask int32 [n,k][, ids_keep, ids_restore])."""
    import torch
    from .engine import default_engine
    eng = default_engine(device)
    st = torch.from_numpy(np.asarray(states, np.uint64).view(np.int64)).to(eng.device)
    n, N_, k = len(st), spec.tokens, spec.masked_count
    mask = torch.empty((n, k), dtype=torch.int32, device=eng.device)
    keep = torch.empty((n, N_ - k), dtype=torch.int64, device=eng.device) if want_ids else None
    rest = torch.empty((n, N_), dtype=torch.int64, device=eng.device) if want_ids else None
    N.check(N.lib().essl_mask_from_states(eng._ctx, N.ptr(st), n, N_, k, N.ptr(mask),
                                          N.ptr(keep), N.ptr(rest), eng._st()),
            "essl_mask_from_states")
    return (mask, keep, rest) if want_ids else mask


def sample_mask(rng, spec: MaskSpec, device=None) -> np.ndarray:
    """Masked token ids, sorted (masking.py:48-56).  Advances ``rng`` exactly as
    the reference shuffle does (tokens - 1 draws)."""
    mask = sample_masks([rng.state], spec, device)[0].cpu().numpy()
    # the shuffle consumed tokens-1 draws of the counter-based stream
    import ctypes
    rng._state = ctypes.c_uint64((rng.state + max(spec.tokens - 1, 0) * _GAMMA) & _M64)
    return mask


def mask_for_epoch(rng, scheme: ScheduleScheme, epoch: int, total_epochs: int,
                   patch: int) -> np.ndarray:
    """masking.py:59-65."""
    p = params_for_epoch(scheme, epoch, total_epochs)
    return sample_mask(rng, MaskSpec.from_resolution(p.resolution, patch, p.masking_ratio))
