"""SplitMix64 streams: the reproducibility contract shared with the reference.

Weight init, batch order and synthetic data must be bit-identical to the
reference so that both implementations see the same inputs. The algorithm
is Vigna's SplitMix64 (constants below); substreams and domains follow
`pkg/src/parconv/rng.py:22-117`:

* ``derive(seed, domain, index)`` = SplitMix64(mix(mix(seed ^ domain*G) ^ index))
* Box-Muller pairs (cos, sin) with u1 = (top53 + 1) * 2^-53, u2 = top53 * 2^-53
* Fisher-Yates from the top index down with ``below(n) = next % n``.

The generator is counter based (output i = mix(state + i*G)), which is what
lets the vectorised array draws here equal the reference's scalar draws.
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB

DOMAIN_INIT = 1
DOMAIN_SHUFFLE = 2
DOMAIN_TEMPLATE = 3
DOMAIN_TRAIN = 4
DOMAIN_TEST = 5
DOMAIN_DROPOUT = 6   # extension: dropout keep masks

_U = np.uint64


def mix64(z: int) -> int:
    """SplitMix64 finaliser on a Python int."""
    z &= M64
    z = ((z ^ (z >> 30)) * _C1) & M64
    z = ((z ^ (z >> 27)) * _C2) & M64
    return z ^ (z >> 31)


def _mix_vec(s: np.ndarray) -> np.ndarray:
    s = (s ^ (s >> _U(30))) * _U(_C1)
    s = (s ^ (s >> _U(27))) * _U(_C2)
    return s ^ (s >> _U(31))


class SplitMix64:
    __slots__ = ("state",)

    def __init__(self, seed: int):
        self.state = seed & M64

    def next_u64(self) -> int:
        self.state = (self.state + GOLDEN) & M64
        return mix64(self.state)

    def next_u64_array(self, n: int) -> np.ndarray:
        if n <= 0:
            return np.empty(0, dtype=np.uint64)
        with np.errstate(over="ignore"):
            states = _U(self.state) + np.arange(1, n + 1, dtype=np.uint64) * _U(GOLDEN)
            self.state = int(states[-1])
            return _mix_vec(states)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * 2.0**-53

    def below(self, n: int) -> int:
        if n <= 0:
            raise ValueError("below() needs n >= 1")
        return self.next_u64() % n

    def gauss_array(self, shape, std: float = 1.0) -> np.ndarray:
        n = int(np.prod(shape))
        half = (n + 1) // 2
        raw = self.next_u64_array(2 * half)
        top = raw >> _U(11)
        u1 = (top[0::2].astype(np.float64) + 1.0) * 2.0**-53
        u2 = top[1::2].astype(np.float64) * 2.0**-53
        radius = np.sqrt(-2.0 * np.log(u1))
        angle = 2.0 * np.pi * u2
        pairs = np.empty((half, 2), dtype=np.float64)
        pairs[:, 0] = radius * np.cos(angle)
        pairs[:, 1] = radius * np.sin(angle)
        return (pairs.reshape(-1)[:n] * std).reshape(shape)

    def gauss(self) -> float:
        return float(self.gauss_array(1)[0])

    def uniform_array(self, shape, low: float = 0.0, high: float = 1.0) -> np.ndarray:
        n = int(np.prod(shape))
        u = (self.next_u64_array(n) >> _U(11)).astype(np.float64) * 2.0**-53
        return (u * (high - low) + low).reshape(shape)

    def shuffle(self, items: np.ndarray) -> None:
        for i in range(len(items) - 1, 0, -1):
            j = self.below(i + 1)
            items[i], items[j] = items[j], items[i]


def derive(seed: int, domain: int, index: int = 0) -> SplitMix64:
    s = mix64((seed & M64) ^ ((domain * GOLDEN) & M64))
    return SplitMix64(mix64(s ^ (index & M64)))


def permutation(seed: int, epoch: int, n: int) -> np.ndarray:
    """Sample order of one epoch; depends on (seed, epoch) only."""
    order = np.arange(n, dtype=np.int64)
    derive(seed, DOMAIN_SHUFFLE, epoch).shuffle(order)
    return order


def dropout_state(seed: int, step: int, layer: int) -> int:
    """SplitMix64 state of the dropout stream of (seed, training step, layer):
    element i of the dense activation (NCHW flatten, global batch row-major)
    draws u_i = mix(state + (i + 1) * GOLDEN) — counter based, so any slice of
    the activation (a replica's rows, a column's channels) draws independently
    and every plan sees the same mask as the dense single-worker run."""
    return derive(seed, DOMAIN_DROPOUT, ((step & 0xFFFFFFFFFFFF) << 16) | (layer & 0xFFFF)).state


def dropout_threshold(p: float) -> int:
    """keep iff (u >> 11) >= threshold, i.e. uniform(u) >= p with uniform = top53 * 2^-53."""
    import math
    return int(math.ceil(p * 2.0**53))


def dropout_keep(seed: int, step: int, layer: int, index: np.ndarray, p: float) -> np.ndarray:
    """Keep mask (bool) of the dense-activation elements ``index`` (int64)."""
    state = _U(dropout_state(seed, step, layer))
    with np.errstate(over="ignore"):
        u = _mix_vec(state + (np.asarray(index, dtype=np.uint64) + _U(1)) * _U(GOLDEN))
    return (u >> _U(11)) >= _U(dropout_threshold(p))
