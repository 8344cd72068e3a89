"""Counter-based SplitMix64 streams (host side).

Mirror of the reference's stream contract (`pkg/src/memcolor/rng.py:1-17`):
the i-th output of the stream with key K is ``mix64(K + (i+1)*GOLDEN)``
(mod 2^64), ``mix64`` being the SplitMix64 finalizer.  Keys are derived by
chain-hashing (seed, tag, indices...) exactly as ``stream_key`` does
(`rng.py:74-82`).  The device side re-implements the same finalizer in
`csrc/common.cuh`; the validation-mode kernels consume these streams draw for
draw, which is what makes their trajectories bit-exact.

Everything here is vectorised numpy so that population-sized key arrays and
initial colourings (16k x 1000 draws) are produced in milliseconds.
"""

from __future__ import annotations

import numpy as np

MASK64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB

# purpose tags (`rng.py:28-34`); part of the reproducibility contract
TAG_INIT = 0x01
TAG_LS = 0x02
TAG_CROSS = 0x03
TAG_NET_INIT = 0x04
TAG_TRAIN = 0x05
TAG_SELECT = 0x06
TAG_MISC = 0x07

_U_GOLDEN = np.uint64(GOLDEN)
_U_MIX1 = np.uint64(_MIX1)
_U_MIX2 = np.uint64(_MIX2)
_S30, _S27, _S31, _S11 = (np.uint64(s) for s in (30, 27, 31, 11))


def mix64_int(z: int) -> int:
    """SplitMix64 finalizer on a Python int (`rng.py:41-45`)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * _MIX1) & MASK64
    z = ((z ^ (z >> 27)) * _MIX2) & MASK64
    return z ^ (z >> 31)


def mix64(z):
    """Vectorised finalizer on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _S30)) * _U_MIX1
        z = (z ^ (z >> _S27)) * _U_MIX2
    return z ^ (z >> _S31)


def stream_values(key, counters):
    """Outputs ``counters`` of the stream(s) ``key`` (broadcasting uint64)."""
    key = np.asarray(key, dtype=np.uint64)
    ctr = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = key + (ctr + np.uint64(1)) * _U_GOLDEN
    return mix64(z)


def stream_value(key, counter) -> int:
    """Scalar ``stream_value`` (`rng.py:56-59`)."""
    return mix64_int((int(key) + ((int(counter) + 1) * GOLDEN)) & MASK64)


def u64_below(key, counter, n) -> int:
    """Scalar bounded draw ``value % n`` (`rng.py:62-65`)."""
    return stream_value(key, counter) % int(n)


def stream_key(master_seed, tag, *indices) -> int:
    """Chain-hashed key of (seed, tag, indices...) (`rng.py:74-82`)."""
    key = mix64_int((int(master_seed) & MASK64) ^ ((int(tag) * GOLDEN) & MASK64))
    for ix in indices:
        key = mix64_int(key + (int(ix) & MASK64) * GOLDEN + 1)
    return key


def stream_keys(master_seed, tag, generation, count, start=0):
    """``[stream_key(seed, tag, generation, i) for i in start..start+count)]``
    as a uint64 array, vectorised (same chain as `rng.py:74-82`)."""
    base = mix64_int((int(master_seed) & MASK64) ^ ((int(tag) * GOLDEN) & MASK64))
    base = mix64_int(base + (int(generation) & MASK64) * GOLDEN + 1)
    idx = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(base) + idx * _U_GOLDEN + np.uint64(1)
    return mix64(z)


def batch_uniform(key, start_counter, count):
    """Uniforms ``start_counter .. +count-1`` of a stream (`rng.py:85-96`)."""
    v = stream_values(np.uint64(int(key) & MASK64),
                      np.arange(start_counter, start_counter + count, dtype=np.uint64))
    return (v >> _S11) * (1.0 / 9007199254740992.0)


class Stream:
    """Stateful view over a counter-based stream (`rng.py:99-125`)."""

    def __init__(self, key):
        self.key = int(key) & MASK64
        self.counter = 0

    @classmethod
    def derive(cls, master_seed, tag, *indices):
        return cls(stream_key(master_seed, tag, *indices))

    def u64(self):
        v = stream_value(self.key, self.counter)
        self.counter += 1
        return v

    def below(self, n):
        return self.u64() % int(n)

    def uniform(self):
        return (self.u64() >> 11) * (1.0 / 9007199254740992.0)

    def below_many(self, n, count):
        """``count`` consecutive ``below(n)`` draws, vectorised."""
        v = stream_values(np.uint64(self.key),
                          np.arange(self.counter, self.counter + count, dtype=np.uint64))
        self.counter += count
        return v % np.uint64(n)

    def shuffle(self, arr):
        for i in range(len(arr) - 1, 0, -1):
            j = self.below(i + 1)
            arr[i], arr[j] = arr[j], arr[i]
