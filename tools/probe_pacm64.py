"""Phase latency probe of the fp64 PaCM kernel (clock64 marks of CTA 0, first pass):
per weight stage, the wait for its bulk copy and the compute + barrier."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_02361_b200 import _capi, tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device  # noqa: E402

ctx = tt.Context(0)
sk = make_sketch(WORKLOADS["r50_c3x3_64"]())
dev = reference_device()
m = tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
ids = tt.random_init(ctx, sk, 512, 3, with_identity=True)[1]
for _ in range(3):
    m.score(sk, dev, ids, tt.TT_PREC_FP64)
ctx.sync() if hasattr(ctx, "sync") else None
import torch  # noqa: E402
torch.cuda.synchronize()
clk = (C.c_longlong * 24)()
C.CDLL(_capi.LIB_PATH).ttdbg_pacm64_clocks(clk, 24)
c = np.array(clk[:24], dtype=np.int64)
names = ["w1 (24->h, stmt)", "w2 (h->h, stmt)", "we (23->h, block)", "wq", "wk", "wv", "head1a", "head1b"]
print("features load", c[1] - c[0])
prev = c[1]
for s, nm in enumerate(names):
    print(f"stage {s} {nm:18s} wait {c[2 + 2 * s] - prev:6d}  compute+sync {c[3 + 2 * s] - c[2 + 2 * s]:6d}")
    prev = c[3 + 2 * s]
print("attention: QK^T", c[19] - c[13], "softmax", c[20] - c[19], "PV", c[21] - c[20], "concat", c[22] - c[21],
      "| head1a wait after concat", c[14] - c[22], "| tail", c[18] - c[17], "total", c[18] - c[0])
