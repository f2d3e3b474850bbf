"""The sm_100a tcgen05 tile engine (TMA SWIZZLE_128B loads, K-major and MN-major UMMA
descriptors, TMEM accumulators) against a plain fp32 matmul of the same bf16 inputs."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1805_01772_b200 import cf  # noqa: E402


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("bn", [128, 256])
@pytest.mark.parametrize("M,N,K", [(256, 512, 1024), (200, 320, 192), (128, 256, 64)])
def test_tc_gemm(a_mn, b_mn, bn, M, N, K):
    torch.manual_seed(M + N + K + a_mn + 2 * b_mn)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    As = A.t().contiguous() if a_mn else A
    Bs = B.t().contiguous() if b_mn else B
    C = torch.full((M, N), float("nan"), device="cuda")
    cf.debug_tc_gemm(M, N, K, bn, a_mn, b_mn, As, Bs, C)
    ref = A.float() @ B.float().t()
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
