"""The NCCL calls behind se2m_exchange_halo on real hardware (one GPU in this allocation): a one-rank
communicator made by the library sends buffers to itself through ncclGroupStart / ncclSend / ncclRecv /
ncclGroupEnd (se2m_nccl_selftest), with the NCCL the process loaded — PyTorch's bundled copy, as in bench.py's
row-band path."""
import pytest

from paper_2503_02412_b200 import se2map as S


@pytest.mark.gpu
@pytest.mark.parametrize("count", [1, 12345, 1 << 22])
def test_nccl_loopback(count):
    import torch  # noqa: F401  (torch's NCCL is the one dlopen returns, as in the bench process)
    ver = S.nccl_selftest(0, count)
    assert ver >= 21800, ver  # ncclSend / ncclRecv need NCCL >= 2.7; the pool's torch ships 2.28


@pytest.mark.gpu
def test_nccl_selftest_rejects_bad_count():
    with pytest.raises(S.Se2mError):
        S.nccl_selftest(0, 0)
