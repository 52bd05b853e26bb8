"""Timeline of ONE draft+verify round replayed from its CUDA graph (fp64,
r50_c3x3_64, N = 65,536, K = 512): %globaltimer marks of the fused selector
(k_fsel) and the fused verify kernel (k_verify64), against CUDA events
around the round on the context stream. Shows where the round's wall time
goes between and inside the two kernels."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_02361_b200 import _capi, tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device  # noqa: E402

ctx = tt.Context(0)
dev = reference_device()
tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
L = C.CDLL(_capi.LIB_PATH)
for name in sys.argv[1:] or ["r50_c3x3_64"]:
    sk = make_sketch(WORKLOADS[name]())
    soa = tt.random_init(ctx, sk, 65536, 42)
    stream = torch.cuda.current_stream()
    for rep in range(4):
        torch.cuda.synchronize()
        span = (C.c_ulonglong * 7)()
        L.ttdbg_verify64_span(span, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tt.round_async(ctx, sk, dev, 65536, 512, 10, soa=soa)
        e1.record(stream)
        out = tt.round_collect(ctx, 10)
        torch.cuda.synchronize()
    sel = (C.c_ulonglong * 24)()
    L.ttdbg_select_clocks(sel, 24)
    L.ttdbg_verify64_span(span, 0)
    s, v = list(sel), list(span)
    t0 = s[0]
    us = lambda x: (x - t0) / 1e3  # noqa: E731
    print(f"{name}: round (events) {e0.elapsed_time(e1) * 1e3:.1f} us | selector {us(s[0]):.1f} -> {us(s[5]):.1f} | "
          f"verify first CTA start {us(v[0]):.1f}, past wait {us(v[1]):.1f}..{us(v[2]):.1f}, last CTA done "
          f"{us(v[3]):.1f}, finish {us(v[4]):.1f} (ids {us(v[6]):.1f}) -> {us(v[5]):.1f} us")

# ---- back-to-back rounds as the bench runs them (7 subgraphs, lagged collect): gaps between kernels
R50 = ["r50_stem", "r50_c1x1_64", "r50_c3x3_64", "r50_c1x1_256", "r50_c3x3_128", "r50_c3x3_256", "r50_c3x3_512"]
sks = [make_sketch(WORKLOADS[w]()) for w in R50]
pops = [tt.random_init(ctx, s_, 65536, 42) for s_ in sks]
seeded = os.environ.get("SEEDED") == "1"
for rep in range(3):
    inflight = 0
    torch.cuda.synchronize()
    for s_, p_ in zip(sks, pops):
        if seeded:
            tt.round_async(ctx, s_, dev, 65536, 512, 10, seed=42)
        else:
            tt.round_async(ctx, s_, dev, 65536, 512, 10, soa=p_)
        inflight += 1
        if inflight > 1:
            tt.round_collect(ctx, 10)
            inflight -= 1
    tt.round_collect(ctx, 10)
    torch.cuda.synchronize()
st = (C.c_ulonglong * 128)()
vt = (C.c_ulonglong * 128)()
ns, nv = C.c_uint(0), C.c_uint(0)
L.ttdbg_select_timeline(st, C.byref(ns))
L.ttdbg_verify64_timeline(vt, C.byref(nv))
S_ = [(st[2 * ((ns.value - 7 + q) % 64)], st[2 * ((ns.value - 7 + q) % 64) + 1]) for q in range(7)]
V_ = [(vt[2 * ((nv.value - 7 + q) % 64)], vt[2 * ((nv.value - 7 + q) % 64) + 1]) for q in range(7)]
t0 = S_[0][0]
print("last step (7 rounds), us from the first selector start:")
for q in range(7):
    print(f"  round {q}: selector {(S_[q][0]-t0)/1e3:7.1f} -> {(S_[q][1]-t0)/1e3:7.1f} | verify {(V_[q][0]-t0)/1e3:7.1f} -> "
          f"{(V_[q][1]-t0)/1e3:7.1f}" + (f" | gap to next selector {(S_[q+1][0]-V_[q][1])/1e3:5.1f}" if q < 6 else ""))
