import ctypes as C, numpy as np, torch
from paper_2402_02361_b200 import tiletune as tt
from tests import _refs as R
n, b = 5000, 4
ctx = tt.Context(0)
for kind in ["pos", "neg", "normal"]:
    if kind == "pos": s = np.array([(i * 7919 % 1000) / 10.0 for i in range(n)])
    elif kind == "neg": s = np.array([((i * 7919 % 1000) - 500) / 100.0 for i in range(n)])
    else: s = np.round(np.random.default_rng(1).normal(size=n), 2)
    d = np.array([(i % 13) / 10.0 for i in range(n)])
    got = tt.select_top(ctx, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), None, b)
    print(kind, got, R.O_select_top(s, d, None, b))
