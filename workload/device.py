"""The generator of ``workload/__init__.py`` re-expressed in torch int64 ops, so
the same keys and queries can be drawn where they are used: on the GPU
(BASELINE.json configs 4-5 need 2^30 keys per rank; drawing and sorting them
with numpy on the host would take minutes and 8 GB of host memory per rank).

Bit-identical to the numpy generator by construction and by test
(``tests/test_workload.py::test_device_generator_matches_numpy``, on torch's
CPU backend here and on CUDA in ``tests/test_gpu_workload.py``).  Like the
numpy module it holds none of the method's arithmetic: it draws numbers.

Unsigned 64-bit values live in int64 tensors as bit patterns:
* wrapping add / multiply / xor are the same bits as on uint64;
* logical right shift = arithmetic shift, then mask the sign-extended bits;
* unsigned order = signed order after flipping bit 63 (``_flip``);
* unsigned ``x mod n`` = ``((x >>> 1) mod n * 2 + (x & 1)) mod n`` (no overflow
  for n < 2^62).
u32 keys are int32 tensors carrying the 32-bit patterns.
"""
from __future__ import annotations

import torch

from . import GOLDEN, MASK64, KEY_SEED, QUERY_SEED, stream_base, splitmix64_int  # noqa: F401

_SIGN = -(1 << 63)          # int64 bit pattern of 1 << 63


def _s64(x: int) -> int:
    """Python int (mod 2^64) -> the int64 with the same bits."""
    x &= MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _flip(x: torch.Tensor) -> torch.Tensor:
    """int64 bits -> int64 whose signed order is the unsigned order of x."""
    return x ^ _SIGN


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 bit patterns (wrapping)."""
    z = x + _s64(GOLDEN)
    z = (z ^ _lsr(z, 30)) * _s64(0xBF58476D1CE4E5B9)
    z = (z ^ _lsr(z, 27)) * _s64(0x94D049BB133111EB)
    return z ^ _lsr(z, 31)


def hash_stream(seed: int, stream: int, start: int, count: int, device) -> torch.Tensor:
    """h(seed, stream, i) for i in [start, start+count), int64 bit patterns."""
    base = stream_base(seed, stream)
    i = torch.arange(count, dtype=torch.int64, device=device) + _s64(base + start)
    return splitmix64(i)


def _to_width(v: torch.Tensor, key_bytes: int) -> torch.Tensor:
    """u64 draw -> key of the width, as an int64 holding the unsigned value
    (u32: the top 32 bits)."""
    if key_bytes == 8:
        return v
    if key_bytes == 4:
        return _lsr(v, 32)
    raise ValueError("key_bytes must be 4 or 8")


def _sorted_unique(v: torch.Tensor, key_bytes: int) -> torch.Tensor:
    if key_bytes == 8:
        s = _flip(torch.sort(_flip(v)).values)
    else:
        s = torch.sort(v).values            # u32 values are non-negative in int64
    return torch.unique_consecutive(s)


def _narrow(v: torch.Tensor, key_bytes: int) -> torch.Tensor:
    """int64 holding unsigned keys -> the storage dtype (int64 / int32 bits)."""
    if key_bytes == 8:
        return v
    return torch.where(v >= (1 << 31), v - (1 << 32), v).to(torch.int32)


def _widen(k: torch.Tensor) -> torch.Tensor:
    """storage dtype -> int64 holding the unsigned key."""
    if k.dtype == torch.int64:
        return k
    return k.to(torch.int64) & 0xFFFFFFFF


def gen_keys(n: int, key_bytes: int = 8, seed: int = KEY_SEED, device="cuda") -> torch.Tensor:
    """n unique, uniformly drawn w-bit unsigned keys, ascending (unsigned
    order), as int64 (u64) or int32 (u32) bit patterns on `device`.  Same
    numbers as ``workload.gen_keys``."""
    if n < 1:
        raise ValueError("n must be >= 1")
    w = 8 * key_bytes
    if n > (1 << w):
        raise ValueError("n exceeds the key domain")
    draw = n + (2 * n * n >> w) + 64
    got = _sorted_unique(_to_width(hash_stream(seed, 0, 0, draw, device), key_bytes), key_bytes)
    pos = draw
    while got.numel() < n:
        extra = max(n - got.numel(), 1) * 2 + 64
        more = _to_width(hash_stream(seed, 0, pos, extra, device), key_bytes)
        pos += extra
        got = _sorted_unique(torch.cat([got, more]), key_bytes)
    if got.numel() > n:
        # keep the n candidates with the smallest independent hash of their value
        # (numpy: argpartition(r, n-1)[:n]; hash values are distinct in practice)
        salt = _s64(stream_base(seed, 3))
        r = _flip(splitmix64(got ^ salt))
        drop = torch.topk(r, got.numel() - n, largest=True, sorted=False).indices
        keep = torch.ones(got.numel(), dtype=torch.bool, device=got.device)
        keep[drop] = False
        got = got[keep]
    return _narrow(got.contiguous(), key_bytes)


def _umod(x: torch.Tensor, n: int) -> torch.Tensor:
    if n & (n - 1) == 0:
        return x & (n - 1)
    return (torch.remainder(_lsr(x, 1), n) * 2 + (x & 1)) % n


def gen_queries(keys: torch.Tensor, m: int, seed: int = QUERY_SEED, hit_ratio: float = 1.0,
                order: str = "random", start: int = 0, chunk: int = 1 << 26) -> torch.Tensor:
    """Slice [start, start+m) of the query stream for `seed`, on keys' device
    (same numbers as ``workload.gen_queries``)."""
    n = keys.numel()
    kb = keys.element_size()
    dev = keys.device
    out = torch.empty(m, dtype=keys.dtype, device=dev)
    thr = None
    if hit_ratio < 1.0:
        thr = min(int(max(hit_ratio, 0.0) * 2.0 ** 64), MASK64)
    for c0 in range(0, m, chunk):
        c = min(chunk, m - c0)
        idx = _umod(hash_stream(seed, 1, start + c0, c, dev), n)
        q = keys[idx]
        if thr is not None:
            is_hit = _flip(hash_stream(seed, 2, start + c0, c, dev)) < _s64(thr ^ (1 << 63))
            miss = _narrow(_to_width(hash_stream(seed, 4, start + c0, c, dev), kb), kb)
            q = torch.where(is_hit, q, miss)
        out[c0:c0 + c] = q
    if order == "sorted":
        out = sort_unsigned(out)
    elif order != "random":
        raise ValueError("order must be 'random' or 'sorted'")
    return out


def sort_unsigned(x: torch.Tensor) -> torch.Tensor:
    """Ascending unsigned order of int64 / int32 bit patterns."""
    if x.dtype == torch.int64:
        return _flip(torch.sort(_flip(x)).values)
    return _narrow(torch.sort(_widen(x)).values, 4)


def gen_keys_range(n: int, lo: int, hi: int, seed: int, shard: int, device="cuda") -> torch.Tensor:
    """n unique u64 keys uniform in [lo, hi) (BASELINE config 5: shard s of a
    range-partitioned key set draws from its own value range), ascending, as
    int64 bit patterns.  Draws h(seed, 16 + shard, i) * (hi - lo) >> 64 + lo
    (multiply-high: uniform for a power-of-two width), dedupes, tops up."""
    width = hi - lo
    if not (0 < width <= (1 << 64)) or width & (width - 1):
        raise ValueError("range width must be a power of two")
    if n > width:
        raise ValueError("n exceeds the range")
    sh = 64 - (width.bit_length() - 1)
    got = None
    pos = 0
    while got is None or got.numel() < n:
        # over-draw by twice the expected duplicates plus slack (as gen_keys)
        extra = (n + (2 * n * n >> (width.bit_length() - 1)) + 64) if got is None else (n - got.numel()) * 2 + 64
        v = hash_stream(seed, 16 + shard, pos, extra, device)
        pos += extra
        if sh == 64:
            v = torch.zeros_like(v)
        elif sh > 0:
            v = _lsr(v, sh)
        v = v + _s64(lo)
        got = v if got is None else torch.cat([got, v])
        got = _flip(torch.unique(_flip(got)))      # sorted unique in unsigned order
    if got.numel() > n:
        # a uniform n-subset: drop the candidates with the largest independent hash
        r = _flip(splitmix64(got ^ _s64(stream_base(seed, 3))))
        drop = torch.topk(r, got.numel() - n, largest=True, sorted=False).indices
        keep = torch.ones(got.numel(), dtype=torch.bool, device=got.device)
        keep[drop] = False
        got = got[keep]
    return got.contiguous()
