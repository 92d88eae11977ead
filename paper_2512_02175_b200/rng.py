"""Counter-based random streams (reference ``graphsde/rng.py``).

Draw ``k`` of stream ``i`` under ``seed`` is the reference's
Philox4x32-10 word ``raw64(seed, i, k)`` (``rng.py:45-66``); uniforms are
``(r >> 11) 2^-53`` and normals the AS241 quantile on the centred lattice
(``rng.py:69-149``).  The scalar functions evaluate the same
``__host__ __device__`` code the kernels use, through ``libgsde.so``.
"""

from __future__ import annotations

from . import _native


def raw64(seed: int, stream: int, index: int) -> int:
    return int(_native.lib().gsde_raw64(seed, stream, index))


def u64_to_uniform(r: int) -> float:
    """``(r >> 11) 2^-53`` in [0, 1) (``rng.py:69-72``)."""
    return float(_native.lib().gsde_u64_to_uniform(int(r) & 0xFFFFFFFFFFFFFFFF))


def norm_ppf(p: float) -> float:
    """Standard normal quantile, AS241 with the far-tail Newton polish
    (``rng.py:81-134``)."""
    return float(_native.lib().gsde_norm_ppf(float(p)))


def u64_to_normal(r: int) -> float:
    """Normal variate of a raw word, on the centred 53-bit lattice
    (``rng.py:137-143``)."""
    return float(_native.lib().gsde_u64_to_normal(int(r) & 0xFFFFFFFFFFFFFFFF))


def uniform01(seed: int, stream: int, index: int) -> float:
    return float(_native.lib().gsde_uniform01(seed, stream, index))


def normal(seed: int, stream: int, index: int) -> float:
    return float(_native.lib().gsde_normal(seed, stream, index))


class RngStream:
    """Stateful cursor over one particle's stream (reference ``rng.py:152-174``)."""

    __slots__ = ("seed", "particle", "counter")

    def __init__(self, seed: int, particle: int = 0, counter: int = 0):
        self.seed = int(seed)
        self.particle = int(particle)
        self.counter = int(counter)

    def uniform(self) -> float:
        u = uniform01(self.seed, self.particle, self.counter)
        self.counter += 1
        return u

    def normal(self) -> float:
        w = normal(self.seed, self.particle, self.counter)
        self.counter += 1
        return w
