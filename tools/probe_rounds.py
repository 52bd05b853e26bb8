"""Per-subgraph round latency (explicit population and seeded), to spot selector retries."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2402_02361_b200 import tiletune as tt
from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device

R50 = ["r50_stem", "r50_c1x1_64", "r50_c3x3_64", "r50_c1x1_256", "r50_c3x3_128", "r50_c3x3_256", "r50_c3x3_512"]
ctx = tt.Context(0)
dev = reference_device()
tt.PaCM(ctx, tt.init_params(64, derive_seed(42, TAG_INIT)), 64)
for name in R50:
    sk = make_sketch(WORKLOADS[name]())
    soa = tt.random_init(ctx, sk, 65536, 42)
    for mode in ("soa", "seeded"):
        ts = []
        for rep in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            out = (tt.draft_verify_round(ctx, sk, dev, 65536, 512, 10, soa=soa, precision=1) if mode == "soa" else
                   tt.draft_verify_round(ctx, sk, dev, 65536, 512, 10, seed=42, precision=1))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"{name:14s} {mode:6s} status={out.status} drafted={out.drafted} rescored={out.rescored} us: "
              + " ".join(f"{t:.0f}" for t in ts))
