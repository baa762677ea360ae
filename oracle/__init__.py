"""CPU oracle for batched sorted-array point lookups (arXiv 2506.01576).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2506_01576_b200`` never imports it and
shares no code with it.

* ``oracle.c`` (loaded here through ctypes) is the plain definition of what
  every variant of the method returns: the unsigned lower bound plus an explicit
  miss bit (readings R1, R3, R4, R20).
* ``oracle.replay`` follows the paper's own algorithms step by step (Listing 1,
  §4.2 pinning with Listing 2's corrected mapping, §5 K-ary search) for small
  cases; it exists to pin the paper's worked examples, not to produce
  expected values for the GPU.

Parity status: every function here is pinned by tests/test_oracle.py and
tests/test_replay.py (brute force, numpy.searchsorted, the invariant
a[lb-1] < q <= a[lb], PAPER.md worked examples in tests/golden/).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (no CUDA involved)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-Wall", "-shared", "-fPIC", "-o", tmp, _SRC, "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            u64 = ctypes.c_uint64
            vp = ctypes.c_void_p
            lib.oracle_lower_bound_u64.argtypes = [vp, u64, u64]
            lib.oracle_lower_bound_u64.restype = u64
            lib.oracle_lower_bound_u32.argtypes = [vp, u64, ctypes.c_uint32]
            lib.oracle_lower_bound_u32.restype = u64
            lib.oracle_lookup.argtypes = [vp, u64, ctypes.c_int, vp, u64, vp, ctypes.c_int]
            lib.oracle_lookup.restype = ctypes.c_int
            lib.oracle_lookup_mt.argtypes = [vp, u64, ctypes.c_int, vp, u64, vp, ctypes.c_int, ctypes.c_int]
            lib.oracle_lookup_mt.restype = ctypes.c_int
            _lib = lib
    return _lib


def miss_bit(out_bytes: int) -> int:
    return 1 << (8 * out_bytes - 1)


def lower_bound(keys: np.ndarray, q: int) -> int:
    """lb(q) = #{i : a[i] < q}, unsigned (oracle.c)."""
    keys = np.ascontiguousarray(keys)
    lib = _load()
    if keys.dtype == np.uint64:
        return int(lib.oracle_lower_bound_u64(keys.ctypes.data, keys.size, int(q)))
    if keys.dtype == np.uint32:
        return int(lib.oracle_lower_bound_u32(keys.ctypes.data, keys.size, int(q)))
    raise TypeError("keys must be uint32 or uint64")


def lookup(keys: np.ndarray, queries: np.ndarray, out_bytes: int | None = None,
           threads: int = 1) -> np.ndarray:
    """out[i] = lb(q_i) if a[lb] == q_i else lb | MISS_BIT (oracle.c)."""
    keys = np.ascontiguousarray(keys)
    queries = np.ascontiguousarray(queries)
    if keys.dtype not in (np.uint32, np.uint64) or queries.dtype != keys.dtype:
        raise TypeError("keys/queries must share dtype uint32 or uint64")
    kb = keys.dtype.itemsize
    ob = kb if out_bytes is None else out_bytes
    out = np.empty(queries.size, dtype={4: np.uint32, 8: np.uint64}[ob])
    lib = _load()
    if threads <= 1:
        rc = lib.oracle_lookup(keys.ctypes.data, keys.size, kb, queries.ctypes.data, queries.size,
                               out.ctypes.data, ob)
    else:
        rc = lib.oracle_lookup_mt(keys.ctypes.data, keys.size, kb, queries.ctypes.data, queries.size,
                                  out.ctypes.data, ob, int(threads))
    if rc != 0:
        raise ValueError("oracle_lookup rejected its arguments (n == 0, or out_bytes=4 with n >= 2^31)")
    return out
