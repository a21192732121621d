"""Find which device-generated C5 member breaks the batched kernel; save it."""
import subprocess, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1710_00125_b200 import gallery

if len(sys.argv) > 1 and sys.argv[1] == "one":
    from paper_1710_00125_b200 import FactorConfig, batched
    a = torch.from_numpy(np.load(sys.argv[2])).cuda()[None]
    cfg = FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=0)
    bf = batched.factor_batched_device(a, cfg, check=False)
    torch.cuda.synchronize()
    print("ok", bf.stats)
    sys.exit(0)
a = gallery.c5_batch_device(16, 256, seed=1).cpu().numpy()
import os
os.makedirs("gpurun_out", exist_ok=True)
for i in range(16):
    fn = f"gpurun_out/c5m_{i}.npy"
    np.save(fn, a[i])
    r = subprocess.run([sys.executable, __file__, "one", fn], capture_output=True, text=True, timeout=120)
    print(i, "sym", np.array_equal(a[i], a[i].T), "rc", r.returncode, r.stdout.strip()[-200:], r.stderr.strip()[-150:])
