import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1710_00125_b200 import api, gallery, _native
n = 32768
a = gallery.type6(n, 0)
an = torch.from_numpy(a).pin_memory().numpy()
cfg = api.FactorConfig(b=128, q=128, p=144, seed=0)
lib = _native.load()
orig = lib.rcp_factor_dist
box = {}
def wrapped(*args):
    t = time.perf_counter(); r = orig(*args); box["c"] = time.perf_counter() - t; return r
lib.rcp_factor_dist = wrapped
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = T(); f = api.factor(an, cfg); t1 = T()
    print(f"api.factor {1e3*(t1-t0):.0f} ms; C call {1e3*box['c']:.0f} ms")
t = T(); om = np.random.Generator(np.random.Philox(0)).standard_normal((144, n)); print("omega draw ms", 1e3*(time.perf_counter()-t))
ad = torch.from_numpy(an).cuda()
for rep in range(2):
    t0 = T(); df = api.factor_device(ad, cfg); t1 = T(); h = df.to_host(); t2 = T()
    print(f"factor_device {1e3*(t1-t0):.0f} ms (C call {1e3*box['c']:.0f}, device {df.stats['t_factor_ms']:.0f}); to_host {1e3*(t2-t1):.0f} ms")
