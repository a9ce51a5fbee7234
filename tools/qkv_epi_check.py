"""QKV projection GEMM (config 2: M = 118784, N = 960, K = 320): the V^T split epilogue
(EPI_SPLIT_VT, what attention consumes) against a plain channels-last store of all 960
columns -- the cost of transposing V in the epilogue."""
import ctypes as C
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_09253_b200 import _lib
from paper_2501_09253_b200._dev import stream

M, N, K, D = 118784, 960, 320, 320
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") / 18).to(torch.bfloat16)
qk = torch.empty(M, 2 * D, device="cuda", dtype=torch.bfloat16)
vt = torch.empty(D, M, device="cuda", dtype=torch.bfloat16)
full = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)


def run(epi):
    g = _lib.GemmArgs()
    g.a, g.lda, g.M, g.a_mode = a.data_ptr(), K, M, 0
    g.b, g.N, g.K = b.data_ptr(), N, K
    if epi == 3:
        g.epi, g.out, g.ldo, g.out2, g.ldo2, g.n_split = 3, qk.data_ptr(), 2 * D, vt.data_ptr(), M, 2 * D
    else:
        g.epi, g.out, g.ldo = 0, full.data_ptr(), N
    _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))


for epi in (3, 0, 3, 0):
    for _ in range(3):
        run(epi)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run(epi)
    e1.record()
    torch.cuda.synchronize()
    print(f"epi={epi}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
