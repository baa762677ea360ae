"""Thin ctypes binding of libbs.so (include/bs.h) — argument marshalling only.

Every step of the lookup path runs in the library's CUDA kernels; this module
only converts torch tensors / numpy arrays to pointers and status codes to
exceptions.  It fails loudly (ImportError / BsError) when the library is
missing: there is no CPU fallback.

Function names follow the C ABI: bs_layout_default, bs_build, bs_lookup,
bs_lookup_ex, bs_lookup_host, bs_destroy, bs_index_info, bs_export,
bs_last_error, bs_version, bs_dist_*.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BS_LIB_PATH: another build of the same library (A/B timing runs in tools/)
LIB_PATH = os.environ.get("BS_LIB_PATH") or os.path.join(_HERE, "lib", "libbs.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "bs.h")

BS_OK, BS_ERR_INVALID, BS_ERR_UNSUPPORTED, BS_ERR_OOM, BS_ERR_CUDA, BS_ERR_NCCL, BS_ERR_NOT_SORTED = 0, -1, -2, -3, -4, -5, -6
NAIVE, OPT, KARY = 0, 1, 2
DYNAMIC, STATIC = 0, 1
REORDER_NONE, REORDER_LOOKUP, REORDER_FULL, REORDER_SORTED, REORDER_GLOBAL, REORDER_BUCKET = 0, 1, 2, 3, 4, 5
HINT_STREAM_EVICT_FIRST, HINT_LEAF_EVICT_FIRST, HINT_SEP_EVICT_LAST = 1, 2, 4
EXPORT_SORTED, EXPORT_PINNED, EXPORT_KARY = 0, 1, 2
DIST_REPLICATED, DIST_PARTITIONED = 0, 1
PIN_MAX = 0xFFFFFFFF

_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64


class bs_layout(ctypes.Structure):
    _fields_ = [(f, _u32) for f in (
        "struct_size", "key_bytes", "out_bytes", "input_sorted", "variant", "schedule", "threads", "nreg",
        "pin_bytes", "pin_partial", "reorder", "k", "leaf_chunk", "ctas_per_sm", "cache_hints", "kary_mode")] + [
        ("reserved", _u32 * 6)]


class bs_launch(ctypes.Structure):
    _fields_ = [(f, _u32) for f in (
        "struct_size", "variant", "schedule", "threads", "nreg", "reorder", "pin_partial", "ctas_per_sm",
        "cache_hints", "use_pinned", "kary_mode")] + [("reserved", _u32 * 5)]


class bs_info(ctypes.Structure):
    _fields_ = [("struct_size", _u32), ("key_bytes", _u32), ("out_bytes", _u32), ("n", _u64),
                ("footprint_bytes", _u64), ("array_bytes", _u64), ("pinned_entries", _u64),
                ("pinned_levels", _u32), ("pinned_partial", _u32), ("search_levels", _u32),
                ("kary_levels", _u32), ("k", _u32), ("leaf_chunk", _u32), ("node_slots", _u32),
                ("kary_smem_levels", _u32), ("separator_slots", _u64), ("separator_bytes", _u64),
                ("build_ms", ctypes.c_double), ("sm_count", _u32), ("smem_per_cta_opt", _u32),
                ("smem_per_cta_kary", _u32), ("build_stage_us", _u32 * 5)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "build_stage_us"}
        d["build_stage_us"] = list(self.build_stage_us)
        return d


class BsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libbs status {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libbs.so (built by paper_2506_01576_b200/build.py). Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i = ctypes.c_void_p, ctypes.c_int
        L.bs_layout_default.argtypes = [ctypes.POINTER(bs_layout)]
        L.bs_launch_default.argtypes = [vp, ctypes.POINTER(bs_launch)]
        L.bs_build.argtypes = [vp, _u64, ctypes.POINTER(bs_layout), ctypes.POINTER(vp)]
        L.bs_lookup.argtypes = [vp, vp, _u64, vp, vp]
        L.bs_lookup_ex.argtypes = [vp, vp, _u64, vp, vp, ctypes.POINTER(bs_launch)]
        L.bs_lookup_host.argtypes = [vp, vp, _u64, vp, vp]
        L.bs_lookup_ws.argtypes = [vp, vp, _u64, vp, vp, ctypes.POINTER(bs_launch), vp, _u64]
        L.bs_workspace_bytes.argtypes = [vp, _u64, ctypes.POINTER(bs_launch), ctypes.POINTER(_u64)]
        L.bs_destroy.argtypes = [vp]
        L.bs_destroy.restype = None
        L.bs_last_error.restype = ctypes.c_char_p
        L.bs_version.restype = ctypes.c_char_p
        L.bs_launch_count.restype = _u64
        L.bs_launch_count.argtypes = []
        L.bs_index_info.argtypes = [vp, ctypes.POINTER(bs_info)]
        L.bs_export.argtypes = [vp, i, vp, _u64, ctypes.POINTER(_u64)]
        L.bs_dist_get_uid.argtypes = [vp]
        L.bs_dist_init.argtypes = [vp, i, i, ctypes.POINTER(vp)]
        L.bs_build_dist.argtypes = [vp, vp, _u64, i, ctypes.POINTER(bs_layout), _u64, ctypes.POINTER(vp)]
        L.bs_lookup_dist.argtypes = [vp, vp, _u64, vp, vp]
        L.bs_dist_destroy.argtypes = [vp]
        L.bs_dist_destroy.restype = None
        L.bs_build_peer.argtypes = [vp, _u64, ctypes.POINTER(bs_layout), i, i, _u64, _u64, ctypes.POINTER(vp)]
        L.bs_peer_export.argtypes = [vp, vp]
        L.bs_peer_connect.argtypes = [vp, vp]
        L.bs_lookup_peer.argtypes = [vp, vp, _u64, vp, vp]
        L.bs_peer_status.argtypes = [vp, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(_u64)]
        L.bs_peer_results.argtypes = [vp, ctypes.POINTER(vp)]
        L.bs_merge.argtypes = [vp, vp, _u64, i, ctypes.POINTER(vp)]
        L.bs_erase.argtypes = [vp, vp, _u64, i, ctypes.POINTER(vp)]
        for f in ("bs_layout_default", "bs_launch_default", "bs_build", "bs_lookup", "bs_lookup_ex",
                  "bs_lookup_host", "bs_index_info", "bs_export", "bs_dist_get_uid", "bs_dist_init",
                  "bs_build_dist", "bs_lookup_dist", "bs_build_peer", "bs_peer_export", "bs_peer_connect",
                  "bs_lookup_peer", "bs_peer_status", "bs_peer_results", "bs_merge", "bs_erase",
                  "bs_lookup_ws", "bs_workspace_bytes"):
            getattr(L, f).restype = i
        _lib = L
    return _lib


def header_symbols(path: str = HEADER) -> list[str]:
    """Function names declared in include/bs.h."""
    txt = open(path).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bs_[a-z_0-9]+)\s*\(", txt)))


def _check(rc):
    if rc != BS_OK:
        raise BsError(rc, bs_last_error())
    return rc


def bs_last_error() -> str:
    return lib().bs_last_error().decode()


def bs_version() -> str:
    return lib().bs_version().decode()


def bs_launch_count() -> int:
    return int(lib().bs_launch_count())


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()   # torch.Tensor


def _stream_ptr(stream) -> int:
    if stream is None:
        return 0
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def bs_layout_default(**over) -> bs_layout:
    lay = bs_layout()
    _check(lib().bs_layout_default(ctypes.byref(lay)))
    for k, v in over.items():
        setattr(lay, k, v)
    return lay


class Index:
    """Owns a bs_index handle; bs_destroy on close()/GC."""

    def __init__(self, handle: int, layout: bs_layout):
        self.handle = handle
        self.layout = layout

    def close(self):
        if self.handle:
            lib().bs_destroy(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def info(self) -> dict:
        return bs_index_info(self)


def bs_build(keys, n: int | None = None, layout: bs_layout | None = None) -> Index:
    """keys: CUDA tensor, CPU tensor or numpy array (device or host memory)."""
    if layout is None:
        layout = bs_layout_default()
    if n is None:
        n = keys.numel() if hasattr(keys, "numel") else keys.size
    h = ctypes.c_void_p()
    _check(lib().bs_build(_ptr(keys), n, ctypes.byref(layout), ctypes.byref(h)))
    return Index(h.value, layout)


def bs_launch_default(index: Index) -> bs_launch:
    L = bs_launch()
    _check(lib().bs_launch_default(index.handle, ctypes.byref(L)))
    return L


def bs_lookup(index: Index, queries, m: int, out, stream=None):
    return _check(lib().bs_lookup(index.handle, _ptr(queries), m, _ptr(out), _stream_ptr(stream)))


def bs_lookup_ex(index: Index, queries, m: int, out, stream=None, launch: bs_launch | None = None, **over):
    if launch is None:
        launch = bs_launch_default(index)
    for k, v in over.items():
        setattr(launch, k, v)
    return _check(lib().bs_lookup_ex(index.handle, _ptr(queries), m, _ptr(out), _stream_ptr(stream),
                                     ctypes.byref(launch)))


def _launch(index: Index, launch, over):
    if launch is None:
        launch = bs_launch_default(index)
    for k, v in over.items():
        setattr(launch, k, v)
    return launch


def bs_workspace_bytes(index: Index, m: int, launch: bs_launch | None = None, **over) -> int:
    n = _u64()
    _check(lib().bs_workspace_bytes(index.handle, m, ctypes.byref(_launch(index, launch, over)), ctypes.byref(n)))
    return n.value


def bs_lookup_ws(index: Index, queries, m: int, out, stream=None, ws=None, ws_bytes: int | None = None,
                 launch: bs_launch | None = None, **over):
    """ws: a device buffer (torch tensor) of at least bs_workspace_bytes(...) bytes."""
    if ws_bytes is None:
        ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    return _check(lib().bs_lookup_ws(index.handle, _ptr(queries), m, _ptr(out), _stream_ptr(stream),
                                     ctypes.byref(_launch(index, launch, over)), _ptr(ws), ws_bytes))


def bs_lookup_host(index: Index, host_queries, m: int, host_out, stream=None):
    return _check(lib().bs_lookup_host(index.handle, _ptr(host_queries), m, _ptr(host_out), _stream_ptr(stream)))


def bs_merge(index: Index, delta_keys, m: int, delta_sorted: bool = False) -> Index:
    """New index over index's keys plus m delta keys (device), same layout."""
    h = ctypes.c_void_p()
    _check(lib().bs_merge(index.handle, _ptr(delta_keys), m, 1 if delta_sorted else 0, ctypes.byref(h)))
    return Index(h.value, index.layout)


def bs_erase(index: Index, del_keys, m: int, del_sorted: bool = False) -> Index:
    """New index over index's keys minus every key equal to one of m device keys."""
    h = ctypes.c_void_p()
    _check(lib().bs_erase(index.handle, _ptr(del_keys), m, 1 if del_sorted else 0, ctypes.byref(h)))
    return Index(h.value, index.layout)


def bs_destroy(index: Index):
    index.close()


def bs_index_info(index: Index) -> dict:
    info = bs_info()
    _check(lib().bs_index_info(index.handle, ctypes.byref(info)))
    return info.as_dict()


def bs_export(index: Index, what: int) -> np.ndarray:
    info = bs_index_info(index)
    kb = info["key_bytes"]
    cnt = {EXPORT_SORTED: info["n"], EXPORT_PINNED: info["pinned_entries"],
           EXPORT_KARY: info["separator_slots"]}[what]
    arr = np.empty(max(cnt, 1), dtype={4: np.uint32, 8: np.uint64}[kb])
    wr = _u64()
    _check(lib().bs_export(index.handle, what, arr.ctypes.data, arr.nbytes, ctypes.byref(wr)))
    return arr[: wr.value // kb]


# ---- multi-GPU ----
def bs_dist_get_uid() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().bs_dist_get_uid(buf))
    return buf.raw


def bs_dist_init(uid: bytes, rank: int, world: int) -> int:
    buf = ctypes.create_string_buffer(uid, 128)
    h = ctypes.c_void_p()
    _check(lib().bs_dist_init(buf, rank, world, ctypes.byref(h)))
    return h.value


def bs_build_dist(comm: int, local_keys, n_local: int, mode: int, layout: bs_layout | None, max_m_local: int) -> Index:
    if layout is None:
        layout = bs_layout_default()
    h = ctypes.c_void_p()
    _check(lib().bs_build_dist(comm, _ptr(local_keys), n_local, mode, ctypes.byref(layout), max_m_local,
                               ctypes.byref(h)))
    return Index(h.value, layout)


def bs_lookup_dist(index: Index, local_queries, m_local: int, out_local, stream=None):
    return _check(lib().bs_lookup_dist(index.handle, _ptr(local_queries), m_local, _ptr(out_local),
                                       _stream_ptr(stream)))


def bs_dist_destroy(comm: int):
    lib().bs_dist_destroy(comm)


# ---- fused peer-memory routing (include/bs.h "Fused peer-memory routing") ----
PEER_BLOB_BYTES = 256


def bs_build_peer(local_keys, n_local: int, layout: bs_layout | None, rank: int, world: int, max_m_local: int,
                  recv_capacity: int = 0) -> Index:
    if layout is None:
        layout = bs_layout_default(variant=2, out_bytes=8)
    h = ctypes.c_void_p()
    _check(lib().bs_build_peer(_ptr(local_keys), n_local, ctypes.byref(layout), rank, world, max_m_local,
                               recv_capacity, ctypes.byref(h)))
    return Index(h.value, layout)


def bs_peer_export(index: Index) -> bytes:
    buf = ctypes.create_string_buffer(PEER_BLOB_BYTES)
    _check(lib().bs_peer_export(index.handle, buf))
    return buf.raw


def bs_peer_connect(index: Index, blobs: list[bytes]):
    raw = b"".join(blobs)
    buf = ctypes.create_string_buffer(raw, len(raw))
    return _check(lib().bs_peer_connect(index.handle, buf))


def bs_peer_connect_group(index: Index, group=None):
    """Argument marshalling only: all-gather the blobs over torch.distributed
    (any backend) and connect."""
    import torch.distributed as dist
    blobs = [None] * dist.get_world_size(group)
    dist.all_gather_object(blobs, bs_peer_export(index), group=group)
    return bs_peer_connect(index, blobs)


def bs_lookup_peer(index: Index, local_queries, m_local: int, out_local, stream=None):
    return _check(lib().bs_lookup_peer(index.handle, _ptr(local_queries), m_local, _ptr(out_local),
                                       _stream_ptr(stream)))


def bs_peer_status(index: Index) -> tuple[int, int]:
    err = ctypes.c_uint32()
    calls = _u64()
    _check(lib().bs_peer_status(index.handle, ctypes.byref(err), ctypes.byref(calls)))
    return err.value, calls.value


def bs_peer_results(index: Index) -> int:
    """Device address of this rank's return window (results of the last
    bs_lookup_peer called with out_local=None)."""
    p = ctypes.c_void_p()
    _check(lib().bs_peer_results(index.handle, ctypes.byref(p)))
    return p.value
