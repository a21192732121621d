import subprocess, sys
import numpy as np
import torch
sys.path.insert(0, ".")
if len(sys.argv) > 1:
    from paper_1710_00125_b200 import FactorConfig, batched, gallery
    cnt, src = int(sys.argv[1]), sys.argv[2]
    if src == "np":
        mats = np.stack([gallery.scaled_member(256, s, scaled=(s % 10 == 0)) for s in range(cnt)])
    else:
        mats = np.stack([np.load(f"gpurun_out/c5m_{i % 16}.npy") for i in range(cnt)])
    cfg = FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=0)
    bf = batched.factor_batched_device(torch.from_numpy(mats).cuda(), cfg, check=False)
    torch.cuda.synchronize()
    print("ok", np.bincount(bf.stats["status"]))
    sys.exit(0)
for src in ("dev", "np"):
    for cnt in (2, 3, 8, 16, 40):
        r = subprocess.run([sys.executable, __file__, str(cnt), src], capture_output=True, text=True, timeout=300)
        print(src, cnt, r.returncode, r.stdout.strip()[-80:], r.stderr.strip()[-100:].replace("\n", " "))
