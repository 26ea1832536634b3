"""SplitMix64 streams, bit-compatible with the reference (``rng.py:10-56``).

The device decoder (``csrc/sat_engine.cu``: ``splitmix_*``) computes the same
sequence; this host copy is used by the workload recipes in ``workloads.py``.
A SplitMix64 stream is counter based: the k-th output (k >= 1) of a stream with
initial state s is ``mix(s + k * GOLDEN)``, which is what lets the device
evaluate draws without carrying state between candidates.
"""

from __future__ import annotations

U64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX_M1 = 0xBF58476D1CE4E5B9
MIX_M2 = 0x94D049BB133111EB


def mix64(z: int) -> int:
    """Finaliser of rng.py:13-16."""
    z = ((z ^ (z >> 30)) * MIX_M1) & U64
    z = ((z ^ (z >> 27)) * MIX_M2) & U64
    return z ^ (z >> 31)


class SplitMix64:
    """Same outputs as rng.SplitMix64 (rng.py:20-48)."""

    __slots__ = ("_s",)

    def __init__(self, seed: int):
        self._s = seed & U64

    @property
    def state(self) -> int:
        return self._s

    def next_u64(self) -> int:
        self._s = (self._s + GOLDEN) & U64
        return mix64(self._s)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) / float(1 << 53)

    def below(self, n: int) -> int:
        """Unbiased draw in [0, n): reject r >= 2^64 - (2^64 mod n), else r mod n (rng.py:34-42)."""
        if n <= 0:
            raise ValueError("n must be positive")
        cutoff = (1 << 64) - ((1 << 64) % n)
        r = self.next_u64()
        while r >= cutoff:
            r = self.next_u64()
        return r % n

    def shuffle(self, items: list) -> None:
        """Fisher-Yates from the top index down (rng.py:44-48)."""
        for i in range(len(items) - 1, 0, -1):
            k = self.below(i + 1)
            items[i], items[k] = items[k], items[i]


def substream_state(seed: int, *salts: int) -> int:
    """Initial state of substream(seed, *salts) (rng.py:51-56)."""
    s = seed & U64
    for salt in salts:
        s = mix64(((s ^ (salt & U64)) + GOLDEN) & U64)
    return s


def substream(seed: int, *salts: int) -> SplitMix64:
    return SplitMix64(substream_state(seed, *salts))
