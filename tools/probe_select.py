"""Phase timeline of the fused draft selector k_fsel (%globaltimer marks of
CTA 0, ns): K1, threshold, compact, rank (+ barriers), emit."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import torch
from paper_2402_02361_b200 import tiletune as tt, _capi
from paper_2402_02361_b200.types import WORKLOADS, make_sketch, reference_device

ctx = tt.Context(0)
dev = reference_device()
L = C.CDLL(_capi.LIB_PATH)
round_path = len(sys.argv) > 1 and sys.argv[1] == "round"  # the round's selector (no identities emitted)
if round_path:
    tt.PaCM(ctx, tt.init_params(64, 5), 64)
for name in ["r50_c3x3_64", "gemm1024", "bert_ffn1"]:
    sk = make_sketch(WORKLOADS[name]())
    for n in (65536, 1 << 20, 1 << 24):
        soa = tt.random_init(ctx, sk, n, 42)
        for _ in range(3):
            if round_path:
                tt.draft_verify_round(ctx, sk, dev, n, 512, 10, soa=soa)
            else:
                tt.draft_topk(ctx, sk, dev, soa, 512)
        torch.cuda.synchronize()
        c = (C.c_ulonglong * 24)()
        L.ttdbg_select_clocks(c, 24)
        t = list(c)
        bars = " ".join(f"b{b}: cta0 {(t[8+2*b]-t[0])/1e3:.1f} last {(t[9+2*b]-t[0])/1e3:.1f}" for b in range(3))
        print(f"{name} n={n}: K1 {(t[1]-t[0])/1e3:.1f} us | threshold {(t[2]-t[1])/1e3:.1f} | "
              f"compact {(t[3]-t[2])/1e3:.1f} | rank {(t[4]-t[3])/1e3:.1f} | emit {(t[5]-t[4])/1e3:.1f} | "
              f"total {(t[5]-t[0])/1e3:.1f} us, survivors {t[6]}, attempts {t[7]} | arrivals (us from start) {bars}")
        print(f"   sample loaded {(t[19]-t[1])/1e3:.1f} | emit: start {(t[16]-t[4])/1e3:.1f} dup bits {(t[17]-t[16])/1e3:.1f} "
              f"scan {(t[18]-t[17])/1e3:.1f} write {(t[5]-t[18])/1e3:.1f}")
        del soa
