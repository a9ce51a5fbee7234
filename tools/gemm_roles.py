"""Per-role barrier wait fractions of the config-2 GEMMs (GemmArgs.dbg counters)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2501_09253_b200 import _lib
from paper_2501_09253_b200._dev import stream

T = 118784
def run(name, M, N, K, epi, bn=0, out_tiled=0, a_tiled=0, resid=False, pair=0):
    a = torch.randn(M if not a_tiled else ((M + 127) // 128 * 128), K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.zeros(N, device="cuda")
    dbg = torch.zeros(8, dtype=torch.int64, device="cuda")
    out = torch.empty(max(M * N, (M + 127) // 128 * 128 * N) + 1024, dtype=torch.bfloat16, device="cuda")
    out2 = torch.empty(N * ((M + 63) // 64 * 64), dtype=torch.bfloat16, device="cuda")
    res = torch.randn(M * N, device="cuda").to(torch.bfloat16) if resid else None
    g = _lib.GemmArgs()
    g.a, g.lda, g.M, g.a_mode = a.data_ptr(), K, M, 2 if a_tiled else 0
    g.b, g.N, g.K, g.bias = b.data_ptr(), N, K, bias.data_ptr()
    g.epi, g.out, g.ldo, g.bn, g.out_tiled = epi, out.data_ptr(), N, bn, out_tiled
    g.P, g.ps = M // 1024, 32
    g.cta_pair = pair
    if epi == 3:
        g.out2, g.ldo2, g.n_split, g.ldo = out2.data_ptr(), (M + 63) // 64 * 64, 2 * N // 3, 2 * N // 3
    if epi == 2:
        g.resid, g.c_real = res.data_ptr(), N
    for i in range(3):
        _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(5):
        _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    g.dbg = dbg.data_ptr()
    _lib.check(_lib.load().ps_gemm(stream(), C.byref(g)))
    torch.cuda.synchronize()
    d = dbg.tolist()
    f = lambda a, b: a / b if b else 0
    print(f"{name:8s} {ms*1e3:7.1f} us {2*M*N*K/ms/1e9:7.1f} TF | prod wait {f(d[0],d[1]):.2f} | mma wait-full {f(d[2],d[4]):.2f} wait-acc {f(d[3],d[4]):.2f} | epi wait-acc {f(d[5],d[6]):.2f}")

ONLY = sys.argv[2:] if len(sys.argv) > 2 and sys.argv[1] == "only" else None  # e.g. only conv-ish (for ncu)
_run = run
def run(name, *a, **k):
    if ONLY is None or name in ONLY:
        _run(name, *a, **k)

run("conv-ish", T, 320, 2880, 0)
run("qkv", T, 960, 320, 3)
run("oproj", T, 320, 320, 0)
run("ff1", T, 1280, 320, 1, out_tiled=1)
run("ff2", T, 320, 1280, 2, a_tiled=1, resid=True)
run("ff2-cl", T, 320, 1280, 0, a_tiled=1)
run("plain256", T, 256, 1024, 0)
if len(sys.argv) > 1 and sys.argv[1] == "pair":
    run("conv-p320", T, 320, 2880, 0, bn=320, pair=2)
    run("conv-p160", T, 320, 2880, 0, bn=160, pair=2)
    run("conv-p256", T, 320, 2880, 0, bn=256, pair=2)
    run("conv-s320", T, 320, 2880, 0, bn=320, pair=1)
    run("conv-s160", T, 320, 2880, 0, bn=160, pair=1)
    run("qkv-p", T, 960, 320, 3, pair=2)
    run("oproj-p", T, 320, 320, 0, pair=2)
if len(sys.argv) > 1 and sys.argv[1] == "bn":
    run("ff2-160", T, 320, 1280, 2, a_tiled=1, resid=True, bn=160)
    run("ff2-320", T, 320, 1280, 2, a_tiled=1, resid=True, bn=320)
    run("conv-160", T, 320, 2880, 0, bn=160)
    run("ff1-128", T, 1280, 320, 1, out_tiled=1, bn=128)
    run("qkv-160", T, 960, 320, 3, bn=160)
    run("qkv-128", T, 960, 320, 3, bn=128)
