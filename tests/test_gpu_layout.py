"""Layout fidelity: the structures bs_build materialises, exported to the host,
against the paper's own position formulas (replayed in oracle/replay.py)."""
import numpy as np
import pytest

from oracle import replay

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


def identity_index(n, kb=8, **kw):
    keys = np.arange(n, dtype={4: np.uint32, 8: np.uint64}[kb])
    lay = bs.bs_layout_default(key_bytes=kb, out_bytes=kb, **kw)
    return keys, bs.bs_build(P.as_torch(keys), n, lay)


@pytest.mark.parametrize("n", [14, 100, 1000, 4096, 5000, 65537])
def test_pinned_table_matches_paper_positions(n):
    """the first M steps touch positions n-1-2i*S/2^M; P:121 / Listing 2
    l.24: partial entries of step M+1, largest positions first (reading R9).
    With identity keys the exported table values ARE the positions."""
    keys, idx = identity_index(n, variant=bs.OPT)
    tab = bs.bs_export(idx, bs.EXPORT_PINNED).astype(np.int64)
    assert tab.size == min(n - 1, idx.info["pinned_entries"])
    for budget in (2, 3, 6, 17, 64, 1000, 30000):
        try:
            c = replay.build_pinned_cache(list(range(n)), budget)
        except ValueError:
            continue
        L = len(c.positions)              # includes a[n-1] (footnote 1)
        full = L - 1                      # our table keeps a[n-1] out of the table
        if full + len(c.partial_positions) > tab.size:
            continue
        assert sorted(tab[:full].tolist()) == sorted(set(c.positions) - {n - 1})
        part = tab[full: full + len(c.partial_positions)].tolist()
        assert part == sorted(c.partial_positions, reverse=True)


@pytest.mark.parametrize("n,K,C", [(27, 3, 4), (28, 3, 1), (1000, 17, 16), (4097, 5, 4), (77777, 9, 8), (65536, 33, 32)])
def test_kary_levels_match_replay(n, K, C):
    """§5 separators = chunk maxima, levels top-first, child m*K+j; the
    device layout pads nodes to W = pow2 >= K-1 slots and levels to 128 B."""
    kb = 8
    keys, idx = identity_index(n, kb, variant=bs.KARY, k=K, leaf_chunk=C)
    sep = bs.bs_export(idx, bs.EXPORT_KARY)
    MAX = np.iinfo(np.uint64).max
    want = replay.build_kary(list(range(n)), K, C, sentinel=int(MAX))
    info = idx.info
    W = info["node_slots"]
    assert W >= K - 1 and W & (W - 1) == 0
    assert info["kary_levels"] == len(want)
    align = W if W * kb >= 128 else 128 // kb
    base = 0
    for level in want:
        nodes = len(level) // (K - 1)
        blk = sep[base: base + nodes * W].reshape(nodes, W)
        assert np.array_equal(blk[:, : K - 1].reshape(-1), np.array(level, dtype=np.uint64))
        assert (blk[:, K - 1:] == MAX).all()
        base += nodes * W
        base = (base + align - 1) // align * align
    assert base == sep.size


def test_kary_overhead_paper_value():
    """~3.1 % at K = 17 with 128-B u32 leaves (C = 32): 32800 real separators."""
    n = 1 << 20
    keys, idx = identity_index(n, 4, variant=bs.KARY, k=17, leaf_chunk=32)
    sep = bs.bs_export(idx, bs.EXPORT_KARY)
    real = int((sep != np.iinfo(np.uint32).max).sum())
    # the last separator of the root may equal a[n-1]; every real one is a key
    assert real == replay.kary_separator_count(n, 17, 32) - _sentinel_slots(n, 17, 32)
    assert 0.029 <= replay.kary_separator_count(n, 17, 32) / n <= 0.035


def _sentinel_slots(n, K, C):
    lv = replay.build_kary(list(range(n)), K, C, sentinel=-1)
    return sum(1 for level in lv for s in level if s == -1)
