"""tcgen05 GEMM kernel (gemm_tc.cuh) against a torch fp64 reference of the same product.

Covers both operand precisions (bf16, 3xTF32) and all four operand major-ness combinations
(K-major / MN-major A and B) and N tiles 64/128/256 -- the variants the LSTM path uses for
the input/dx GEMMs (K-major) and the weight-gradient GEMMs (MN-major).
"""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = {0: 2e-2, 1: 5e-6, 2: 5e-6}  # normwise: bf16 operands vs 3xTF32 / fp16x2 (fp32-parity)


def _run(prec, amn, bmn, M, N, K, bn):
    from paper_1604_01946_b200 import _lib
    L = _lib.load()
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K + prec * 11 + amn * 2 + bmn)
    A = torch.randn(M, K, generator=g, dtype=torch.float64)
    B = torch.randn(N, K, generator=g, dtype=torch.float64)
    dA = (A.t() if amn else A).contiguous().float().cuda()
    dB = (B.t() if bmn else B).contiguous().float().cuda()
    lda = M if amn else K
    ldb = N if bmn else K
    dD = torch.zeros(N, M, dtype=torch.float32, device="cuda")  # column-major M x N
    st = L.rw_test_gemm(prec, amn, bmn, M, N, K, dA.data_ptr(), lda, dB.data_ptr(), ldb,
                        dD.data_ptr(), M, bn)
    assert st == 0, L.rw_last_error(None).decode()
    torch.cuda.synchronize()
    ref = (A.float().double() @ B.float().double().t())
    got = dD.t().double().cpu()
    err = (got - ref).norm() / ref.norm()
    return err.item()


@pytest.mark.parametrize("prec,amn,bmn", [(0, 0, 0), (0, 0, 1), (0, 1, 0), (0, 1, 1), (1, 0, 0),
                                           (2, 0, 0), (2, 1, 1)])
def test_gemm_majors(prec, amn, bmn):
    # MN-major operands are used with bf16 only: kind::tf32 reads 32-bit MN-major tiles with a
    # different swizzle atom, so the fp32-parity path feeds K-major (transposed) copies instead
    err = _run(prec, amn, bmn, 256, 256, 512, 128)
    assert err < TOL[prec], err


def test_tf32_mn_major_rejected():
    from paper_1604_01946_b200 import _lib
    L = _lib.load()
    d = torch.zeros(128 * 128, device="cuda")
    assert L.rw_test_gemm(1, 1, 0, 128, 128, 64, d.data_ptr(), 128, d.data_ptr(), 64,
                          d.data_ptr(), 128, 128) == 1


@pytest.mark.parametrize("prec", [0, 1, 2])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_gemm_ntiles(prec, bn):
    if prec != 0 and bn == 256:
        pytest.skip("two-plane formats run 64- or 128-column tiles (2 x 2 bn TMEM columns)")
    err = _run(prec, 0, 0, 128, 2 * bn, 256, bn)
    assert err < TOL[prec], err


def test_gemm_large_k():
    # the weight-gradient shape class: long K (B*T), MN-major operands
    err = _run(0, 1, 1, 512, 256, 6400, 128)
    assert err < TOL[0], err


def test_gemm_large_k_fp32_promotion():
    # fp32-parity at K = 6400: chunked accumulation keeps the error at fp32 level
    err = _run(1, 0, 0, 256, 128, 6400, 64)
    assert err < 2e-6, err
