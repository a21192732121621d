"""Where does the end-to-end factor(numpy) time go at C3?"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1710_00125_b200 import api, gallery
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = gallery.type6(n, 0)
a_pin = torch.from_numpy(a).pin_memory()
an = a_pin.numpy()
cfg = api.FactorConfig(b=128, q=128, p=144, seed=0)
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(2):
    t0 = T()
    ad = torch.from_numpy(np.ascontiguousarray(an)).to("cuda")
    t1 = T()
    df = api.factor_device(ad, cfg)
    t2 = T()
    f = df.to_host()
    t3 = T()
    print(f"rep {rep}: H2D {1e3*(t1-t0):.0f} ms  factor_device {1e3*(t2-t1):.0f} ms (device {df.stats['t_factor_ms']:.0f})  to_host {1e3*(t3-t2):.0f} ms")
    t4 = T()
    g = api.factor(an, cfg)
    t5 = T()
    print(f"   api.factor total {1e3*(t5-t4):.0f} ms")
    del df, f, g, ad
