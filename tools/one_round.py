"""A few draft+verify rounds of one subgraph (a small driver for ncu
captures): python tools/one_round.py [workload] [n] [precision] [reps]"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2402_02361_b200 import tiletune as tt
from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device

name = sys.argv[1] if len(sys.argv) > 1 else "r50_c3x3_64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
prec = tt.TT_PREC_BF16 if (len(sys.argv) > 3 and sys.argv[3] == "bf16") else tt.TT_PREC_FP64
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
ctx = tt.Context(0)
sk = make_sketch(WORKLOADS[name]())
dev = reference_device()
tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
soa = tt.random_init(ctx, sk, n, 42)
for _ in range(reps):
    out = tt.draft_verify_round(ctx, sk, dev, n, 512, 10, soa=soa, precision=prec)
torch.cuda.synchronize()
print(name, n, out.index.tolist())
