"""B200-native batched sorted-array point lookups (arXiv 2506.01576).

The product is libbs.so (C ABI, include/bs.h; CUDA for sm_100a).  This
package holds its sources (csrc/), the in-tree build (build.py) and a thin
ctypes binding (bs.py).  PyTorch is used only for device memory and streams.
"""
from . import bs  # noqa: F401
from .bs import (BsError, Index, bs_build, bs_destroy, bs_export, bs_index_info, bs_last_error,  # noqa: F401
                 bs_launch_default, bs_layout_default, bs_lookup, bs_lookup_ex, bs_lookup_host, bs_version)

_TORCH_VIEW = {4: "int32", 8: "int64"}


def as_torch(arr, device="cuda"):
    """numpy uint32/uint64 -> torch tensor with the same BITS (int32/int64 view).

    torch never orders keys (its int64 would be signed); the library reads the
    memory as unsigned.
    """
    import numpy as np
    import torch
    arr = np.ascontiguousarray(arr)
    t = torch.from_numpy(arr.view(_TORCH_VIEW[arr.dtype.itemsize]))
    return t.to(device) if device != "cpu" else t


def to_numpy_unsigned(t, key_bytes: int):
    import numpy as np
    a = t.detach().cpu().numpy()
    return a.view({4: np.uint32, 8: np.uint64}[key_bytes])
