"""bs_build_dist / bs_lookup_dist on one GPU (world = 1): the NCCL plumbing,
route / scatter / exchange-to-self / add-base / unroute kernels, bit-exact vs
the oracle.  Multi-rank routing math is covered on CPU by test_dist_cpu.py."""
import numpy as np
import pytest

import oracle
import workload

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_01576_b200 as P  # noqa: E402
from paper_2506_01576_b200 import bs  # noqa: E402


@pytest.fixture(scope="module")
def comm():
    uid = bs.bs_dist_get_uid()
    c = bs.bs_dist_init(uid, 0, 1)
    yield c
    bs.bs_dist_destroy(c)


@pytest.mark.parametrize("mode", [bs.DIST_REPLICATED, bs.DIST_PARTITIONED])
@pytest.mark.parametrize("variant", [bs.NAIVE, bs.OPT, bs.KARY])
def test_dist_world1(comm, mode, variant):
    keys = workload.gen_keys(100003, 8, seed=11)
    q = workload.gen_queries(keys, 250001, seed=12, hit_ratio=0.6)
    lay = bs.bs_layout_default(key_bytes=8, out_bytes=8, variant=variant)
    idx = bs.bs_build_dist(comm, P.as_torch(keys), keys.size, mode, lay, q.size)
    out = torch.empty(q.size, dtype=torch.int64, device="cuda")
    bs.bs_lookup_dist(idx, P.as_torch(q), q.size, out)
    torch.cuda.synchronize()
    got = P.to_numpy_unsigned(out, 8)
    assert np.array_equal(got, oracle.lookup(keys, q))
    # m_local = 0 is a valid collective call
    bs.bs_lookup_dist(idx, P.as_torch(q[:1]), 0, out)
    idx.close()


def test_dist_overflow_rejected(comm):
    keys = workload.gen_keys(1000, 8, seed=1)
    idx = bs.bs_build_dist(comm, P.as_torch(keys), keys.size, bs.DIST_PARTITIONED, None, 10)
    q = P.as_torch(workload.gen_queries(keys, 11, seed=2))
    out = torch.empty(11, dtype=torch.int64, device="cuda")
    with pytest.raises(bs.BsError):
        bs.bs_lookup_dist(idx, q, 11, out)


@pytest.mark.parametrize("reorder,n", [(5, 100003), (5, 3 << 20), (4, 100003)])
def test_dist_partitioned_out_of_place_lookup(comm, reorder, n):
    """layout.reorder = BUCKET / GLOBAL: bs_build_dist allocates the workspace for
    its receive capacity and the owner looks the received queries up in that
    mode (as the fused peer path does); several calls reuse it."""
    keys = workload.gen_keys(n, 8, seed=13)
    lay = bs.bs_layout_default(key_bytes=8, out_bytes=8, variant=bs.KARY, reorder=reorder)
    idx = bs.bs_build_dist(comm, P.as_torch(keys), keys.size, bs.DIST_PARTITIONED, lay, 200000)
    out = torch.empty(200000, dtype=torch.int64, device="cuda")
    for call, m in enumerate((200000, 8193, 1)):
        q = workload.gen_queries(keys, m, seed=14 + call, hit_ratio=0.6)
        bs.bs_lookup_dist(idx, P.as_torch(q), m, out)
        torch.cuda.synchronize()
        assert np.array_equal(P.to_numpy_unsigned(out[:m], 8), oracle.lookup(keys, q)), f"call {call}"
    idx.close()
