"""Phase timeline of the fast draft selector (%globaltimer marks, ns)."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import torch
from paper_2402_02361_b200 import tiletune as tt, _capi
from paper_2402_02361_b200.types import WORKLOADS, make_sketch, reference_device

ctx = tt.Context(0)
dev = reference_device()
L = C.CDLL(_capi.LIB_PATH)
for name in ["r50_c3x3_64", "gemm1024", "bert_ffn1"]:
    sk = make_sketch(WORKLOADS[name]())
    for n in (65536, 1 << 20, 1 << 24):
        soa = tt.random_init(ctx, sk, n, 42)
        for _ in range(3):
            tt.draft_topk(ctx, sk, dev, soa, 512)
        torch.cuda.synchronize()
        c = (C.c_ulonglong * 12)()
        L.ttdbg_select_clocks(c, 12)
        t = list(c)
        print(f"{name} n={n}: K1 {(t[1]-t[0])/1e3:.1f} us | threshold {(t[2]-t[1])/1e3:.1f} | gap {(t[3]-t[2])/1e3:.1f} | "
              f"compact {(t[4]-t[3])/1e3:.1f} | rank {(t[5]-t[4])/1e3:.1f} | emit {(t[6]-t[5])/1e3:.1f} | "
              f"total {(t[6]-t[0])/1e3:.1f} us, survivors {t[7]} | emit: zero {(t[8]-t[5])/1e3:.1f} scatter {(t[9]-t[8])/1e3:.1f} scan {(t[10]-t[9])/1e3:.1f} out-loop {(t[11]-t[10])/1e3:.1f} tail {(t[6]-t[11])/1e3:.1f}")
        del soa
