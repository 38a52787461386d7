"""GPU parity of the tcgen05 GEMM behind the LM-head backward (dart_gemm_bf16):
C (+)= A_op B_op^T for K-major and MN-major operands, checked against the
oracle's float64 product (oracle.lmhead_logits = A B^T).  Integer operands
make every fp32 partial sum exact, so fp32 results must match bit for bit
and bf16 results must equal the round-to-nearest-even of the exact value."""
import numpy as np
import pytest
import torch

from oracle import dart_oracle as O
from paper_2509_23866_b200 import dart

pytestmark = pytest.mark.gpu


def _ints(shape, lo, hi, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(lo, hi + 1, shape, generator=g).to(torch.bfloat16)


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K", [(296, 520, 200), (128, 256, 64), (1000, 264, 1032)])
def test_gemm_exact_all_majors(a_mn, b_mn, M, N, K):
    A = _ints((M, K), -3, 3, 1)                     # A_op [M, K]
    B = _ints((N, K), -3, 3, 2)                     # B_op [N, K]
    ref = O.lmhead_logits(A.float().numpy(), B.float().numpy())
    Ad = (A.t().contiguous() if a_mn else A).cuda()
    Bd = (B.t().contiguous() if b_mn else B).cuda()
    C = torch.full((M, N), float("nan"), device="cuda")
    dart.gemm_bf16(Ad, Bd, C, a_mn_major=a_mn, b_mn_major=b_mn)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy().astype(np.float64), ref)
    # accumulate: C += A B^T
    dart.gemm_bf16(Ad, Bd, C, a_mn_major=a_mn, b_mn_major=b_mn, mode=dart.GEMM_ACCUM_F32)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy().astype(np.float64), 2 * ref)
    # bf16 output = RNE of the exact value
    Cb = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    dart.gemm_bf16(Ad, Bd, Cb, a_mn_major=a_mn, b_mn_major=b_mn, mode=dart.GEMM_STORE_BF16)
    torch.cuda.synchronize()
    assert torch.equal(Cb.cpu(), torch.from_numpy(ref).to(torch.bfloat16))


def test_gemm_padded_pitches_and_gaussian():
    """Row pitches larger than the logical width, Gaussian operands: within
    the fp32 accumulation bound (ceil(K/16) + 4) u sum_k |a_k b_k|."""
    M, N, K = 257, 392, 520
    g = torch.Generator().manual_seed(5)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, generator=g).to(torch.bfloat16)                  # stored MN-major (B_op = B.T)
    As = torch.zeros(M, K + 24, dtype=torch.bfloat16); As[:, :K] = A
    Bs = torch.zeros(K, N + 40, dtype=torch.bfloat16); Bs[:, :N] = B
    Cs = torch.zeros(M, N + 8, device="cuda")
    dart.gemm_bf16(As.cuda()[:, :K], Bs.cuda()[:, :N], Cs[:, :N], b_mn_major=True)
    torch.cuda.synchronize()
    ref = O.lmhead_logits(A.float().numpy(), B.float().numpy().T)
    bound = (-(-K // 16) + 4) * 2.0 ** -24 * (np.abs(A.float().numpy()) @ np.abs(B.float().numpy()))
    assert np.all(np.abs(Cs[:, :N].cpu().numpy() - ref) <= bound)
    assert torch.all(Cs[:, N:] == 0)


def test_gemm_rejects_bad_arguments():
    A = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    C = torch.zeros(64, 60, device="cuda")                                   # N % 8 != 0
    with pytest.raises(dart.DartError):
        dart.gemm_bf16(A, A[:60], C)


def test_gemm_store_mode_must_match_c_dtype():
    """The ABI sees only C's pointer: an fp32 store into a bf16 buffer would
    run past its end, so the binding refuses a mode that does not match C's
    dtype and, by default, picks the store mode from it."""
    A = torch.ones(128, 64, dtype=torch.bfloat16, device="cuda")
    Cb = torch.zeros(128, 256, dtype=torch.bfloat16, device="cuda")
    Cf = torch.zeros(128, 256, device="cuda")
    with pytest.raises(dart.DartError):
        dart.gemm_bf16(A, A.new_ones(256, 64), Cb, mode=dart.GEMM_STORE_F32)
    with pytest.raises(dart.DartError):
        dart.gemm_bf16(A, A.new_ones(256, 64), Cf, mode=dart.GEMM_STORE_BF16)
    dart.gemm_bf16(A, A.new_ones(256, 64), Cb)                                # inferred: bf16 store
    dart.gemm_bf16(A, A.new_ones(256, 64), Cf)                                # inferred: fp32 store
    torch.cuda.synchronize()
    assert torch.all(Cb == 64) and torch.all(Cf == 64)
