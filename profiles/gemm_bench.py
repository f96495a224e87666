"""Microbenchmark of the tcgen05 GEMM kernel (gemm_tc.cuh) on the LSTM path's shapes, next to
torch.matmul (cuBLAS) on the same problem for context. Usage: python profiles/gemm_bench.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RW_TEST_GEMM_REPS", "20")
from paper_1604_01946_b200 import _lib  # noqa: E402

L = _lib.load()
SHAPES = [  # (name, prec, a_mn, b_mn, M, N, K, bn)
    ("wgrad dW (4H x I x BT), MN/MN", 0, 1, 1, 2048, 512, 6400, 128),
    ("wgrad dW bn256", 0, 1, 1, 2048, 512, 6400, 256),
    ("dx0 (I x BT x 4H), K/K", 0, 0, 0, 512, 6400, 2048, 256),
    ("dx0 bn128", 0, 0, 0, 512, 6400, 2048, 128),
    ("square 4096^3 K/K", 0, 0, 0, 4096, 4096, 4096, 256),
    ("tf32x3 wgrad K/K", 1, 0, 0, 2048, 512, 6400, 64),
    ("config E wgrad one layer K/K", 0, 0, 0, 8192, 4096, 25600, 256),
    ("config E wgrad one layer K/K bn128", 0, 0, 0, 8192, 4096, 25600, 128),
    ("square 8192^3 K/K", 0, 0, 0, 8192, 8192, 8192, 256),
    ("config E wgrad dR MN/MN bn256", 0, 1, 1, 8192, 2048, 25600, 256),
    ("config E wgrad dR MN/MN bn128", 0, 1, 1, 8192, 2048, 25600, 128),
    ("config C2048 wgrad dR MN/MN bn256", 0, 1, 1, 8192, 2048, 12800, 256),
]
if os.environ.get("GEMM_ONLY"):
    SHAPES = [s for s in SHAPES if os.environ["GEMM_ONLY"] in s[0]]
out = []
for name, prec, amn, bmn, M, N, K, bn in SHAPES:
    A = torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")
    B = torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")
    D = torch.zeros(N, M, device="cuda")
    st = L.rw_test_gemm(prec, amn, bmn, M, N, K, A.data_ptr(), M if amn else K, B.data_ptr(),
                        N if bmn else K, D.data_ptr(), M, bn)
    ms = L.rw_test_gemm_last_ms() if st == 0 else float("nan")
    a16 = A.to(torch.bfloat16)
    b16 = B.to(torch.bfloat16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        (a16.t() if amn else a16) @ (b16 if bmn else b16.t())
    e0.record()
    for _ in range(20):
        (a16.t() if amn else a16) @ (b16 if bmn else b16.t())
    e1.record()
    torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) / 20
    tf = 2 * M * N * K / (ms * 1e-3) / 1e12
    out.append(dict(name=name, ms=ms, tflops=tf, cublas_bf16_ms=cub,
                    cublas_tflops=2 * M * N * K / (cub * 1e-3) / 1e12, status=st))
    print(json.dumps(out[-1]), flush=True)
