import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1710_00125_b200 import FactorConfig, batched, gallery
n, cnt = int(sys.argv[1]), int(sys.argv[2])
mats = np.stack([gallery.scaled_member(n, s, scaled=(s % 2 == 1)) for s in range(cnt)])
bf = batched.factor_batched_device(torch.from_numpy(mats).cuda(), FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=0),
                                   check=False)
torch.cuda.synchronize()
st = bf.stats
print("status", np.unique(st["status"], return_counts=True))
bad = np.nonzero(st["status"] == 98)[0]
for i in bad[:10]:
    print("matrix", i, "mask", st["num_kind"][i], "step", st["num_step"][i])
