"""Small batched factor run (for compute-sanitizer)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1710_00125_b200 import FactorConfig, batched, gallery

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mats = np.stack([gallery.scaled_member(n, s, scaled=(s % 2 == 1)) for s in range(cnt)])
bf = batched.factor_batched_device(torch.from_numpy(mats).cuda(), FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=0),
                                   check=False)
torch.cuda.synchronize()
print(bf.stats["status"], bf.stats["n_steps"])
