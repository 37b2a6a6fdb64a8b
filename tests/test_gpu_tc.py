"""tcgen05 plumbing (TMA, 128B swizzle, UMMA descriptors, TMEM) vs torch fp32."""

import pytest
import torch

from paper_2210_15748_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("da,db", [(torch.float16, torch.float16), (torch.bfloat16, torch.bfloat16)])
@pytest.mark.parametrize("M,N", [(128, 256), (300, 224), (64, 16), (1000, 112)])
def test_tc_selftest_matches_fp32(da, db, M, N):
    g = torch.Generator(device="cuda").manual_seed(M * N)
    A = torch.randn(M, 128, device="cuda", generator=g).to(da)
    B = torch.randn(N, 128, device="cuda", generator=g).to(db)
    D = engine.tc_selftest(A, B)
    ref = A.double() @ B.double().T
    err = (D.double() - ref).abs().max().item()
    assert err < 1e-3, err
