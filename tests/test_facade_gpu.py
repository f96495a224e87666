"""GPU: the C++ drop-in facade (include/rnnwave/engine.hpp) used the way the reference's own
tests use rnnwave::Engine (tests/cpp/facade_parity.cpp), checked against the C restatement
of the reference with the SURVEY §8c tolerances."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_facade_parity():
    exe = os.path.join(HERE, "cpp", "build", "facade_parity")
    if not os.path.exists(exe):
        subprocess.run(["sh", os.path.join(HERE, "cpp", "build.sh")], check=True, capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout[-6000:])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "FACADE PASS" in out.stdout


def test_reference_harness_through_facade():
    """The reference's OWN acceptance code (verify.hpp check_determinism, check_cross_level,
    the LSTM draws of check_oracle_agreement, and sched::validate_trace over the device trace)
    compiled unmodified against the facade (tests/cpp/reference_harness.cpp). The binary is built
    where the reference sources exist (tests/cpp/build.sh) and travels to the GPU box."""
    exe = os.path.join(HERE, "cpp", "build", "reference_harness")
    if not os.path.exists(exe):
        pytest.skip("reference_harness not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(out.stdout[-6000:])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "ALL PASS" in out.stdout


def test_device_gemm_matches_fp64():
    """rw_gemm (the facade's gemm, gemm.hpp:339-347 semantics) against a float64 product for
    every transpose combination, ragged sizes, alpha / beta and leading dimensions > rows."""
    import ctypes as C
    import numpy as np
    from paper_1604_01946_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(3)
    F = C.POINTER(C.c_float)
    for ta in (0, 1):
        for tb in (0, 1):
            M, N, K = 37, 70, 129
            A = np.asfortranarray(rng.standard_normal((K, M) if ta else (M, K) ).astype(np.float32))
            Bm = np.asfortranarray(rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32))
            Cbig = np.asfortranarray(rng.standard_normal((M + 5, N)).astype(np.float32))
            C0 = Cbig.copy(order="F")
            alpha, beta = 0.75, -0.5
            st = L.rw_gemm(ta, tb, M, N, K, alpha, A.ctypes.data_as(F), A.shape[0], Bm.ctypes.data_as(F),
                           Bm.shape[0], beta, Cbig.ctypes.data_as(F), M + 5)
            assert st == 0, L.rw_last_error(None).decode()
            opA = A.T if ta else A
            opB = Bm.T if tb else Bm
            ref = alpha * (opA.astype(np.float64) @ opB.astype(np.float64)) + beta * C0[:M].astype(np.float64)
            err = np.linalg.norm(Cbig[:M] - ref) / np.linalg.norm(ref)
            assert err < 5e-6, (ta, tb, err)
            assert np.array_equal(Cbig[M:], C0[M:])  # rows past M untouched
