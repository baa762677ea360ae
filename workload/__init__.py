"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no search, no lower bound,
no encoding).  It only draws numbers.  Both sides of every parity test receive
the arrays produced here; the oracle never sees anything produced by the CUDA
library and vice versa.

Recipe (§2, P:61 — "2^26 unique and
uniformly-drawn 32-bit unsigned integers ... probes 2^27 uniformly-drawn keys
from the build set in random order"):

* ``h(seed, stream, i) = splitmix64(base(seed, stream) + i)`` — counter-based,
  so any slice of a stream can be regenerated independently (per-rank shards).
* keys: a uniform n-subset (without replacement) of the w-bit unsigned domain,
  returned ascending (unsigned order; numpy sorts uint32/uint64 unsigned).
* hits: ``keys[h(seed_q, 1, j) mod n]`` — uniform draws from the build set WITH
  replacement (m = 2n forces replacement).
* misses (hit_ratio < 1): uniform w-bit values ``h(seed_q, 4, j)``; such a
  value coincides with a key with probability n / 2^w, in which case it is
  simply a hit.  The realised hit count is whatever the oracle says.
* order: "random" (as drawn) or "sorted" (ascending, the Fig. 1b workload).
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

# Measured-run seeds.
KEY_SEED = 20250601
QUERY_SEED = 20250602

_CHUNK = 1 << 24


def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser over a uint64 array (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix64_int(x: int) -> int:
    """Scalar splitmix64 on Python ints (for stream bases)."""
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def stream_base(seed: int, stream: int) -> int:
    return splitmix64_int(seed & MASK64) ^ splitmix64_int((stream * 0x632BE59BD9B4E019 + 1) & MASK64)


def hash_stream(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """h(seed, stream, i) for i in [start, start+count) as uint64."""
    base = stream_base(seed, stream)
    with np.errstate(over="ignore"):
        idx = np.arange(count, dtype=np.uint64) + np.uint64((base + start) & MASK64)
    return splitmix64(idx)


def _to_width(v: np.ndarray, key_bytes: int) -> np.ndarray:
    if key_bytes == 8:
        return v.astype(np.uint64, copy=False)
    if key_bytes == 4:
        return (v >> np.uint64(32)).astype(np.uint32)
    raise ValueError("key_bytes must be 4 or 8")


def _sorted_unique(v: np.ndarray) -> np.ndarray:
    """np.unique without its slow path (numpy 2.3 takes ~26 s for 2^24 u64):
    sort, then drop repeats.  Same result, ascending."""
    s = np.sort(v)
    if s.size < 2:
        return s
    keep = np.empty(s.size, dtype=bool)
    keep[0] = True
    np.not_equal(s[1:], s[:-1], out=keep[1:])
    return s[keep]


def key_dtype(key_bytes: int):
    return {4: np.uint32, 8: np.uint64}[key_bytes]


def gen_keys(n: int, key_bytes: int = 8, seed: int = KEY_SEED) -> np.ndarray:
    """n unique, uniformly drawn w-bit unsigned keys, ascending."""
    if n < 1:
        raise ValueError("n must be >= 1")
    w = 8 * key_bytes
    if n > (1 << w):
        raise ValueError("n exceeds the key domain")
    # expected duplicate fraction ~ n / 2^(w+1): over-draw by twice that plus slack
    draw = n + (2 * n * n >> w) + 64
    got = _sorted_unique(_to_width(hash_stream(seed, 0, 0, draw), key_bytes))
    pos = draw
    while got.size < n:
        extra = max(n - got.size, 1) * 2 + 64
        more = _to_width(hash_stream(seed, 0, pos, extra), key_bytes)
        pos += extra
        got = _sorted_unique(np.concatenate([got, more]))
    if got.size > n:
        # keep a uniform n-subset: rank every candidate by an independent hash
        # of its own value (independent of draw order), keep the n smallest.
        salt = np.uint64(stream_base(seed, 3))
        r = splitmix64(got.astype(np.uint64) ^ salt)
        keep = np.sort(np.argpartition(r, n - 1)[:n])
        got = got[keep]
    return np.ascontiguousarray(got)


def gen_queries(keys: np.ndarray, m: int, seed: int = QUERY_SEED, hit_ratio: float = 1.0,
                order: str = "random", start: int = 0) -> np.ndarray:
    """m lookup keys; slice [start, start+m) of the query stream for `seed`."""
    keys = np.asarray(keys)
    n = keys.shape[0]
    kb = keys.dtype.itemsize
    out = np.empty(m, dtype=keys.dtype)
    if hit_ratio >= 1.0:
        thr = None
    else:
        thr = np.uint64(min(int(max(hit_ratio, 0.0) * 2.0 ** 64), MASK64))
    for c0 in range(0, m, _CHUNK):
        c = min(_CHUNK, m - c0)
        idx = hash_stream(seed, 1, start + c0, c) % np.uint64(n)
        q = keys[idx]
        if thr is not None:
            is_hit = hash_stream(seed, 2, start + c0, c) < thr
            miss = _to_width(hash_stream(seed, 4, start + c0, c), kb)
            q = np.where(is_hit, q, miss)
        out[c0:c0 + c] = q
    if order == "sorted":
        out.sort()
    elif order != "random":
        raise ValueError("order must be 'random' or 'sorted'")
    return out


def adversarial_queries(keys: np.ndarray, seed: int = 1, extra: int = 64) -> np.ndarray:
    """Every key, plus below-min / above-max / 0 / MAX / gap values.

    Gap values are key+1 and key-1 (wrapping avoided), which are absent unless
    adjacent keys exist — the oracle decides.
    """
    keys = np.asarray(keys)
    dt = keys.dtype
    mx = np.iinfo(dt).max
    parts = [keys, np.array([0, 1, mx, mx - 1], dtype=dt)]
    if keys.size:
        lo = keys[keys > 0] - dt.type(1)
        hi = keys[keys < mx] + dt.type(1)
        parts += [lo, hi]
    r = _to_width(hash_stream(seed, 5, 0, extra), dt.itemsize)
    parts.append(r)
    q = np.concatenate(parts).astype(dt)
    perm = np.argsort(hash_stream(seed, 6, 0, q.size), kind="stable")
    return np.ascontiguousarray(q[perm])
