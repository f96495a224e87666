"""One tcgen05 GEMM through rw_test_gemm against a torch fp32 reference of bf16-rounded inputs
(scaled max error and kernel time). Usage: python profiles/gemm2_debug.py M N K a_mn b_mn [bn]
(bn 256 with > 148 tiles selects the CTA-pair kernel k_gemm_p2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1604_01946_b200 import _lib
L = _lib.load()
M, N, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
amn, bmn = int(sys.argv[4]), int(sys.argv[5])
bn = int(sys.argv[6]) if len(sys.argv) > 6 else 256
torch.manual_seed(0)
A = torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")
B = torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")
D = torch.zeros(N, M, device="cuda")
st = L.rw_test_gemm(0, amn, bmn, M, N, K, A.data_ptr(), M if amn else K, B.data_ptr(), N if bmn else K, D.data_ptr(), M, bn)
torch.cuda.synchronize()
Ab = (A.t() if amn else A).to(torch.bfloat16).float()
Bb = (B.t() if bmn else B).to(torch.bfloat16).float()
ref = Ab @ Bb.t()
err = (D.t() - ref).abs().max().item() / ref.abs().max().item()
print("status", st, "scaled max err", err, "ms", L.rw_test_gemm_last_ms())
