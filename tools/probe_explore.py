"""One explore at TunerConfig defaults, for ncu launch lists (tools only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_02361_b200 import tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import WORKLOADS, make_sketch, reference_device  # noqa: E402

ctx = tt.Context(0)
sk = make_sketch(WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "gemm1024"]())
for r in range(2):
    tt.explore(ctx, sk, reference_device(), 32, 512, 512, 7 + r)

# phase marks of the last k_mutate (clock64 of thread 0)
import ctypes as C  # noqa: E402
import numpy as np  # noqa: E402
from paper_2402_02361_b200 import _capi  # noqa: E402
clk = (C.c_longlong * 8)()
C.CDLL(_capi.LIB_PATH).ttdbg_mutate_clocks(clk, 8)
c = np.array(clk[:8], dtype=np.int64)
print("k_explore_gens generation-1 cycles: weights+lengths", c[1] - c[0], "sum || offset chain", c[2] - c[1], "stitch", c[3] - c[2], "apply", c[4] - c[3],
      "| thread 0 of CTA 0: child built", c[5] - c[3], "draft cost", c[6] - c[5], "identity", c[7] - c[6],
      "writes", c[4] - c[7])
