"""Phase latency probe of the tensor-core PaCM kernel (clock64 marks of one tile)."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2402_02361_b200 import tiletune as tt, _capi
from paper_2402_02361_b200.types import WORKLOADS, make_sketch, reference_device, derive_seed, TAG_INIT

ctx = tt.Context(0)
sk = make_sketch(WORKLOADS["r50_c3x3_64"]())
dev = reference_device()
m = tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
L = C.CDLL(_capi.LIB_PATH)
for k in (16, 512, 65536):
    ids = tt.random_init(ctx, sk, k, 3, with_identity=True)[1]
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.score(sk, dev, ids, tt.TT_PREC_BF16)
        e1.record()
        torch.cuda.synchronize()
    clk = (C.c_longlong * 16)()
    L.ttdbg_pacm_tc_clocks(clk, 16)
    c = np.array(clk[:16], dtype=np.int64)
    names = ["start", "mma1", "epi1", "mma2", "epi2a", "epi2b", "attn", "head"]
    print(f"k={k}: score (features + tc) {e0.elapsed_time(e1)*1e3:.1f} us; tile marks:",
          " ".join(f"{names[i]}={c[i]-c[0]}" for i in range(1, 8)))
