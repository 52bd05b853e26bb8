"""Phase probe of the h = 64 throughput PaCM kernel (k_pacm64_h64, or with
`round` the fused features + PaCM kernel k_verify64 inside a draft+verify
round): clock64 marks of CTA 0's first pass, and the %globaltimer span."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_02361_b200 import _capi, tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device  # noqa: E402

ctx = tt.Context(0)
fused = "round" in sys.argv[1:]
sk = make_sketch(WORKLOADS["r50_c3x3_64"]())
dev = reference_device()
m = tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
ids = tt.random_init(ctx, sk, 512, 3, with_identity=True)[1]
pop = tt.random_init(ctx, sk, 65536, 7)
L = C.CDLL(_capi.LIB_PATH)
span = (C.c_ulonglong * 7)()
for _ in range(3):
    torch.cuda.synchronize()
    (L.ttdbg_verify64_span if fused else L.ttdbg_pacm64_h64_span)(span, 1)
    if fused:
        if "soa" in sys.argv[1:]:
            tt.draft_verify_round(ctx, sk, dev, 65536, 512, 10, soa=pop)
        else:
            tt.draft_verify_round(ctx, sk, dev, 65536, 512, 10, seed=7)
    else:
        m.score(sk, dev, ids, tt.TT_PREC_FP64)
torch.cuda.synchronize()
(L.ttdbg_verify64_span if fused else L.ttdbg_pacm64_h64_span)(span, 0)
sp = list(span)
print(f"span (ns): first start -> first past pdl_wait {sp[1]-sp[0]}, -> last past wait {sp[2]-sp[0]}, "
      f"-> last CTA done {sp[3]-sp[0]}" + (f", finish {sp[4]-sp[0]} (ids ready {sp[6]-sp[0]}) -> {sp[5]-sp[0]}" if fused else ""))
clk = (C.c_longlong * 24)()
(L.ttdbg_verify64_clocks if fused else L.ttdbg_pacm64_h64_clocks)(clk, 24)
c = np.array(clk[:24], dtype=np.int64)
d = lambda a, b: int(c[b] - c[a])  # noqa: E731
print(f"staging {d(0, 1)} (index load {d(0, 22)} generate {d(22, 23)} combine {d(23, 19)} factors {d(0, 19)} cand_info {d(19, 20)} sync {d(0, 21)}) | wait W1|We {d(1, 2)} | phase 1 {d(2, 3)} sync {d(2, 4)}")
print(f"wait WA {d(4, 5)} | phase 2: S2 {d(5, 6)} Q {d(5, 16)} K {d(5, 17)} V {d(5, 7)} sync {d(5, 8)}")
print(f"phase 3: head1a wait Hw1 {d(8, 9)} chain {d(9, 10)} | logits+softmax {d(8, 11)} PV+pool {d(11, 12)} | sync {d(8, 13)}")
print(f"phase 5: head1b {d(13, 14)} head2 {d(14, 15)}")
print(f"total {d(0, 15)} cycles")

if fused:
    fc = (C.c_longlong * 8)()
    L.ttdbg_verify64_finish_clocks(fc)
    f = list(fc)
    print(f"finish_block: loads+init {f[0]-f[4]} | warp minima {f[1]-f[0]} | candidates {f[2]-f[1]} | rank {f[3]-f[2]} "
          f"cycles; {f[5]} candidates, bound from warp {f[6]}")
