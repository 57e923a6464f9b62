"""Counter-based per-sample random streams (mirror of cropload/rng.py:1-87),
evaluated by the native host library (include/essl.h essl_rng_*)."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N

DOMAIN_PIPELINE = 0
DOMAIN_MASK = 1
DOMAIN_PERMUTATION = 3
_M64 = (1 << 64) - 1


class SampleRng:
    """Deterministic stream for one (seed, epoch, index, domain) key (rng.py:34-77)."""

    __slots__ = ("_state",)

    def __init__(self, seed: int, epoch: int, index: int, domain: int = DOMAIN_PIPELINE):
        self._state = ctypes.c_uint64(N.lib().essl_rng_init(seed & _M64, epoch & _M64,
                                                            index & _M64, domain & _M64))

    @property
    def state(self) -> int:
        return int(self._state.value)

    def next_u64(self) -> int:
        return int(N.lib().essl_rng_next(ctypes.byref(self._state)))

    def random(self) -> float:
        return float(N.lib().essl_rng_random(ctypes.byref(self._state)))

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.random()

    def randint(self, n: int) -> int:
        return int(N.lib().essl_rng_randint(ctypes.byref(self._state), n))

    def shuffle(self, items) -> None:
        for i in range(len(items) - 1, 0, -1):
            j = self.randint(i + 1)
            items[i], items[j] = items[j], items[i]


def epoch_permutation(seed: int, epoch: int, n: int) -> np.ndarray:
    """Visiting order of sample indices for one epoch (rng.py:80-87), C++."""
    out = np.empty(n, np.int64)
    N.check(N.lib().essl_epoch_permutation(seed & _M64, epoch & _M64, n, N.ptr(out)),
            "essl_epoch_permutation")
    return out


def shard(perm: np.ndarray, rank: int, world_size: int, mode: str = "pad") -> np.ndarray:
    """DDP partition of an epoch permutation, rank r taking
    every world_size-th entry from position r:

    - ``"pad"`` (default, torch DistributedSampler semantics): the
      permutation is extended by wrapping to a multiple of world_size first,
      so every rank gets ceil(n / world) samples and the same number of
      batches (no rank waits in a collective on an extra last batch); the
      first few samples of the epoch are seen twice;
    - ``"drop"``: truncated to a multiple of world_size (DistributedSampler
      drop_last), every rank gets floor(n / world);
    - ``"stride"``: plain perm[r::world], an exact partition whose shard
      lengths differ by up to one.
    With world_size == 1 all three are the whole permutation."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank/world_size {rank}/{world_size}")
    n = len(perm)
    if mode == "pad" and n % world_size:
        total = -(-n // world_size) * world_size
        perm = np.concatenate([perm, np.resize(perm, total - n)]) if n else perm
    elif mode == "drop":
        perm = perm[:n - n % world_size]
    elif mode not in ("pad", "stride"):
        raise ValueError(f"shard mode must be pad, drop or stride, got {mode!r}")
    return perm[rank::world_size]


def shard_len(n: int, rank: int, world_size: int, mode: str = "pad") -> int:
    """len(shard(perm of n, rank, world_size, mode)) without building it."""
    if mode == "pad":
        return -(-n // world_size)
    if mode == "drop":
        return n // world_size
    return max(0, (n - rank + world_size - 1) // world_size)
