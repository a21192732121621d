"""Time the batched C5 kernel (device-resident stack) for N matrices: python tools/c5_timing.py [N]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1710_00125_b200 import api, batched, gallery  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cfg = api.FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=0)
a = gallery.c5_batch_device(count, 256, seed=1000, device="cuda")
normals = torch.from_numpy(batched.normal_stream(cfg, 256)).cuda()
ws = torch.empty(batched.batched_workspace_bytes(256, cfg), dtype=torch.uint8, device="cuda")
out = None
best = 1e9
for it in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = batched.factor_batched_device(a, cfg, normals=normals, workspace=ws, out=out, check=False)
    e1.record()
    torch.cuda.synchronize()
    if it:
        best = min(best, e0.elapsed_time(e1))
bad = int((out.stats["status"] != 0).sum())
print(f"C5 {count} matrices: {best:.2f} ms -> {best * 65536 / count:.1f} ms per 65536; "
      f"{count * 256 ** 3 / 3 / (best * 1e-3) / 1e12:.3f} TF; failed {bad}", flush=True)
