"""Single-CTA vs CTA-pair GEMM tiles on the config-2 GEMM shapes: agreement and time."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_09253_b200 import _lib
from paper_2501_09253_b200._dev import stream

T = 118784


def run(name, M, N, K, epi, out_tiled=0, a_tiled=0, resid=False, m_map=None):
    torch.manual_seed(0)
    a = torch.randn(M if not a_tiled else ((M + 127) // 128 * 128), K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda") * 0.1
    res = torch.randn(M * N, device="cuda").to(torch.bfloat16) if resid else None
    outs, times = [], []
    for pair in (1, 2):
        out = torch.zeros(max(M * N, (M + 127) // 128 * 128 * N) + 1024, dtype=torch.bfloat16, device="cuda")
        out2 = torch.zeros(N * ((M + 63) // 64 * 64), dtype=torch.bfloat16, device="cuda")
        g = _lib.GemmArgs()
        g.a, g.lda, g.M, g.a_mode = a.data_ptr(), K, M, 2 if a_tiled else 0
        g.b, g.N, g.K, g.bias = b.data_ptr(), N, K, bias.data_ptr()
        g.epi, g.out, g.ldo, g.bn, g.out_tiled = epi, out.data_ptr(), N, 0, out_tiled
        g.P, g.ps, g.cta_pair = M // 1024, 32, pair
        if m_map is not None:
            g.m_map, g.m_count = m_map.data_ptr(), m_map.numel()
        if epi == 3:
            g.out2, g.ldo2, g.n_split, g.ldo = out2.data_ptr(), (M + 63) // 64 * 64, 2 * N // 3, 2 * N // 3
        if epi == 2:
            g.resid, g.c_real = res.data_ptr(), N
        for i in range(3):
            _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(10):
            _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 10)
        outs.append((out.clone(), out2.clone()))
    same = torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    d = (outs[0][0].float() - outs[1][0].float()).abs().max().item()
    fl = 2 * (M if m_map is None else m_map.numel() * 128) * N * K
    print(f"{name:8s} single {times[0]*1e3:7.1f} us {fl/times[0]/1e9:7.1f} TF | pair {times[1]*1e3:7.1f} us "
          f"{fl/times[1]/1e9:7.1f} TF | identical={same} maxdiff={d:.3g}", flush=True)


run("qkv", T, 960, 320, 3)
run("oproj", T, 320, 320, 0)
run("ff1", T, 1280, 320, 1, out_tiled=1)
run("ff2", T, 320, 1280, 2, a_tiled=1, resid=True)
run("ff2-cl", T, 320, 1280, 0, a_tiled=1)
run("k2880", T, 320, 2880, 0)
mm = torch.arange(0, 928, 3, dtype=torch.int32, device="cuda")  # odd count compaction map
run("mapped", T, 320, 1280, 0, m_map=mm)
run("odd-M", 1000, 192, 320, 0)
