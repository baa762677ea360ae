"""Step-by-step replays of the paper's algorithms (small inputs, pure Python).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  These functions follow
PAPER.md in its own order and notation so a reader can check them by eye; they
exist to pin the paper's worked examples (Fig. 3, Fig. 5, Fig. 7, Fig. 9, the
3.1 % overhead) and to show that each variant lands on the plain lower bound
computed by ``oracle.c``.  They are never used to produce expected values for
the CUDA path — parity tests compare against ``oracle.lookup``.

Readings of garbled passages (DESIGN.md §"Readings"):
  R1  Listing 1: ``step >>= 1`` runs every iteration, not only when
      the step is taken (§3 prose: "the step width is halved in each
      iteration").
  R2  ``bs(buffer, offset, step)`` reads ``sorted_keys``/``lookup`` from the
      enclosing scope; here the signature is (keys, q, offset, step).
  R6  pinned positions n-1-2i*S/2^M -> stride S/2^(M-1).
  R7  footnote 1: the never-probed a[n-1] occupies a cache slot.
  R9  partial (step M+1) entries: largest positions first (Listing 2 l.24).
  R10 Listing 2 l.25-27 adjust offset/step BEFORE the global mapping (l.29-31)
      which overwrites them; the evident intent is applied AFTER mapping, in
      global units.
  R11 Listing 2 l.33 ``bs(cached_keys, ...)`` is read as ``bs(sorted_keys, ...)``.
  R16 K-ary separators are chunk maxima (Fig. 9's exact values cannot be
      reconciled with one spacing rule).
"""
from __future__ import annotations

from dataclasses import dataclass, field


def lpow2(n: int) -> int:
    """LPOW2(n): largest power of two <= n ("count-leading-zeros")."""
    if n < 1:
        raise ValueError("LPOW2 is defined for n >= 1")
    return 1 << (n.bit_length() - 1)


def bs(keys, q, offset: int, step: int, probes: list | None = None) -> int:
    """Listing 1 lines 1-7 with reading R1/R2.

    while step > 0: if step <= offset and keys[offset-step] >= q: offset -= step;
    step >>= 1 (every iteration).
    """
    while step > 0:
        if step <= offset:
            p = offset - step
            if probes is not None:
                probes.append(p)
            if keys[p] >= q:
                offset = p
        step >>= 1
    return offset


def naive(keys, q, probes: list | None = None) -> int:
    """Listing 1 lines 9-13: offset = n-1, step = LPOW2(n)."""
    n = len(keys)
    return bs(keys, q, n - 1, lpow2(n), probes)


def to_lower_bound(keys, q, offset: int) -> int:
    """The loop's clamp: offset points at the first entry >= q, or n-1 if none."""
    return offset if keys[offset] >= q else len(keys)


# ---------------------------------------------------------------- §4.2 pinning

@dataclass
class PinnedCache:
    """SPEC.md PinnedCache; Listing 2's cached_keys / cached_partial_keys / cache_step_size."""
    M: int
    stride: int                      # cache_step_size = S / 2^(M-1)
    positions: list = field(default_factory=list)          # ascending global positions (L)
    partial_positions: list = field(default_factory=list)  # ascending global positions (P)
    cached_keys: list = field(default_factory=list)
    cached_partial_keys: list = field(default_factory=list)


def build_pinned_cache(keys, budget: int) -> PinnedCache:
    """§4.2: the entries of the first M steps sit at positions
    n-1-2i*S/2^M; choose the largest M whose entries fit `budget` slots
    (footnote 1 slot a[n-1] included, R7); fill leftover slots with step-(M+1)
    entries, largest positions first (R9)."""
    n = len(keys)
    if budget < 2 and n > 1:
        raise ValueError("budget_slots must be >= 2")
    S = lpow2(n)
    best = None
    M = 1
    while True:
        stride = (2 * S) >> M            # 2*S / 2^M
        if stride < 1:
            break
        L = (n - 1) // stride + 1
        if L > budget:
            break
        best = (M, stride, L)
        if stride == 1:
            break
        M += 1
    if best is None:
        raise ValueError("budget too small for M = 1")
    M, stride, L = best
    pos = sorted(n - 1 - i * stride for i in range(L))
    partial = []
    if stride >= 2:
        i = 0
        while len(partial) < budget - L:
            p = n - 1 - i * stride - stride // 2
            if p < 0:
                break
            partial.append(p)
            i += 1
    partial = sorted(partial)
    return PinnedCache(M=M, stride=stride, positions=pos, partial_positions=partial,
                       cached_keys=[keys[p] for p in pos],
                       cached_partial_keys=[keys[p] for p in partial])


def search_pinned(keys, cache: PinnedCache, q, full: bool,
                  cache_probes: list | None = None, global_probes: list | None = None) -> int:
    """Listing 2 lines 16-33 with readings R10/R11.

    full=False is BS (steps-pinning), full=True is BS (full-pinning).
    Returns the Listing-1 offset (clamped to n-1 on a miss above the maximum).
    """
    n = len(keys)
    ck = cache.cached_keys
    L = len(ck)
    P = len(cache.cached_partial_keys)
    # l.17-20: binary search in scratch memory
    cprobes: list = []
    offset = bs(ck, q, L - 1, lpow2(L), cprobes)
    if cache_probes is not None:
        cache_probes.extend(n - 1 - (L - 1 - c) * cache.stride for c in cprobes)
    rev_offset = L - 1 - offset                              # l.21
    # l.29-31: global offset
    offset = n - 1 - rev_offset * cache.stride
    step = cache.stride >> 1
    # l.23-27 (R10): the step-(M+1) entry, when cached, is taken from scratch
    if full and rev_offset < P:
        revrev = P - 1 - rev_offset                           # l.24
        if cache_probes is not None:
            cache_probes.append(offset - step)
        if cache.cached_partial_keys[revrev] >= q:            # l.25
            offset -= step                                    # l.26
        step >>= 1                                            # l.27
    # l.33 (R11): continue in the sorted array
    return bs(keys, q, offset, step, global_probes)


# ---------------------------------------------------------------- §4.3 reordering

def block_sort(batch):
    """§4.3: sort a batch; forward[p] = original slot of sorted position p.
    Ties broken by original position (irrelevant to results, R15)."""
    forward = sorted(range(len(batch)), key=lambda i: (batch[i], i))
    return [batch[i] for i in forward], forward


def unsort(results, forward):
    """§4.3 "locally applying the inverse of the sort permutation"."""
    out = [None] * len(results)
    for p, r in enumerate(results):
        out[forward[p]] = r
    return out


# ---------------------------------------------------------------- §5 K-ary search

def build_kary(keys, K: int, C: int, sentinel: int):
    """§5: separators materialised densely, bottom-up, fixed chunk sizes,
    no child pointers; leaf layer = the sorted array.  Separator j of node m at a
    level whose children span `span` keys = max of child m*K+j (R16), sentinel
    (the key type's maximum) for children past the end.  Levels returned
    top-first, each node exactly K-1 wide."""
    if K < 2 or C < 1:
        raise ValueError("K >= 2 and C >= 1 required")
    n = len(keys)
    count = -(-n // C)          # leaf chunks
    span = C
    bottom_up = []
    while count > 1:
        nodes = -(-count // K)
        level = []
        for m in range(nodes):
            for j in range(K - 1):
                child = m * K + j
                if child * span < n:
                    level.append(keys[min((child + 1) * span, n) - 1])
                else:
                    level.append(sentinel)
        bottom_up.append(level)
        span *= K
        count = nodes
    return bottom_up[::-1]


def kary_search(keys, levels, K: int, C: int, q, path: list | None = None) -> int:
    """§5: at each node descend into the first chunk j with
    q <= separator_j (else K-1); search the leaf chunk.  Returns lb in [0, n]."""
    n = len(keys)
    m = 0
    span = C * K ** len(levels)
    for level in levels:
        seps = level[m * (K - 1):(m + 1) * (K - 1)]
        j = next((i for i, s in enumerate(seps) if q <= s), K - 1)
        if path is not None:
            path.append(j)
        m = m * K + j
        span //= K
        if m * span >= n:       # a child past the end: every key is < q
            return n
    lo, hi = m * C, min((m + 1) * C, n)
    for i in range(lo, hi):
        if keys[i] >= q:
            return i
    return hi if hi < n else n


def kary_separator_count(n: int, K: int, C: int) -> int:
    """Total separator slots (sentinels included) of build_kary, in closed form."""
    count = -(-n // C)
    total = 0
    while count > 1:
        nodes = -(-count // K)
        total += nodes * (K - 1)
        count = nodes
    return total
