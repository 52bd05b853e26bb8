"""Stage latency probe of the fp64 PaCM kernel (clock64 marks of one candidate)."""
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
tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
L = C.CDLL(_capi.LIB_PATH)
for k in (1, 20, 512):
    ids = tt.random_init(ctx, sk, k, 3, with_identity=True)[1]
    st, bl = tt.extract_features(ctx, sk, dev, ids)
    m = tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.score_batch(st, bl)
        e1.record()
        torch.cuda.synchronize()
    clk = (C.c_longlong * 24)()
    L.ttdbg_pacm64_clocks(clk, 24)
    c = np.array(clk[:24], dtype=np.int64)
    print(f"k={k}: {e0.elapsed_time(e1)*1e3:.1f} us; marks (cycles from start):")
    names = {1: "W1", 2: "W2", 3: "We", 4: "Wq", 5: "Wk", 6: "Wv", 7: "Hw1a", 8: "Hw1b", 10: "attn", 11: "concat", 21: "end"}
    for i in range(1, 22):
        if c[i]:
            print(f"   {i:2d} {names.get(i, 'wait' + str(i - 12)):8s} {c[i] - c[0]:8d}")
