"""One explore at TunerConfig defaults, for ncu launch lists, plus the
phase marks of one generation of k_explore_gens and a wall-clock split of the
tuner round (tools only): python tools/probe_explore.py [workload]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_02361_b200 import _capi  # noqa: E402
from paper_2402_02361_b200 import tiletune as tt  # noqa: E402
from paper_2402_02361_b200.types import TAG_INIT, WORKLOADS, derive_seed, make_sketch, reference_device  # noqa: E402

ctx = tt.Context(0)
sk = make_sketch(WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "gemm1024"]())
dev = reference_device()
lib = C.CDLL(_capi.LIB_PATH)
for r in range(2):
    tt.explore(ctx, sk, dev, 32, 512, 512, 7 + r)
for pg in (1, 8, 20, 31):
    lib.ttdbg_mutate_probe(pg)
    tt.explore(ctx, sk, dev, 32, 512, 512, 11)
    clk = (C.c_longlong * 26)()
    lib.ttdbg_mutate_clocks(clk, 26)
    c = np.array(clk[:26], dtype=np.int64)
    r = lambda k: int(c[k] - c[0])  # noqa: E731
    print(f"gen {pg}: main: phaseA {r(14)} chain-done {r(22)} staging-done {r(21)} apply {r(3)}..{r(4)} "
          f"[search {r(12) - r(3)} build {r(6) - r(12)} wait-exact {r(8) - r(6)}] "
          f"| prep: start {r(15)} len {r(16)} walks {r(17)} scan {r(18)} rewalk {r(19)} draws {r(20)} "
          f"| sync {r(10)}..{r(11)}", flush=True)
lib.ttdbg_mutate_probe(1)
ns = (C.c_ulonglong * 4)()
lib.ttdbg_mutate_ns(ns)
print(f"kernel: gen-0 phase {ns[1]} ns, whole kernel {ns[2]} ns, {ns[3]} cycles -> {ns[3] / max(ns[2], 1):.3f} GHz")
t0 = time.perf_counter()
for r in range(20):
    tt.explore(ctx, sk, dev, 32, 409, 512, 500 + r, with_soa=False)
print("explore wall ms", round(1e3 * (time.perf_counter() - t0) / 20, 4))
st = (C.c_double * 8)()
lib.ttdbg_explore_stamps(st)
print("host stamps us (entry, flags reset, launched, gen0 seen, gen n-2 seen, last flag, synced, return):",
      [round(x, 1) for x in st])
lib.ttdbg_mutate_ns(ns)
print(f"kernel: gen-0 phase {ns[1]} ns, whole kernel {ns[2]} ns, {ns[3]} cycles -> {ns[3] / max(ns[2], 1):.3f} GHz")

params = tt.init_params(64, derive_seed(5, TAG_INIT))
model = tt.PaCM(ctx, params, 64)
T = {"draft_set": 0.0, "explore": 0.0, "h2d": 0.0, "score": 0.0, "select": 0.0}
reps = 20
for r in range(reps + 2):
    t0 = time.perf_counter()
    tt.explore(ctx, sk, dev, 32, 409, 512, 2000 + r, with_soa=False)
    t1 = time.perf_counter()
    ids, dc, _ = tt.draft_set(ctx, sk, dev, 32, 512, 512, 0.2, 2000 + r, 2001 + r)
    t2 = time.perf_counter()
    ids_d = torch.from_numpy(ids.view(np.int64)).cuda()
    dc_d = torch.from_numpy(dc).cuda()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    sc = model.score(sk, dev, ids_d, tt.TT_PREC_FP64)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    tt.select_top(ctx, sc, dc_d, None, 10)
    t5 = time.perf_counter()
    if r >= 2:
        for k, v in zip(T, (t2 - t1, t1 - t0, t3 - t2, t4 - t3, t5 - t4)):
            T[k] += v / reps
print("tuner round split (ms):", {k: round(1e3 * v, 4) for k, v in T.items()})
t0 = time.perf_counter()
for r in range(reps):
    tt.tuner_round(ctx, sk, dev, 32, 512, 512, 0.2, 3000 + r, 3001 + r, 10)
print("tt_tuner_round ms:", round(1e3 * (time.perf_counter() - t0) / reps, 4))
