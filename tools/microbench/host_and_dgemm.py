"""Probe the GPU box: host CPU/RAM and cuBLAS DGEMM (torch fp64 matmul) throughput."""
import os, subprocess, time, json
import torch
print("cpu:", subprocess.run("lscpu | grep -E 'Model name|^CPU\\(s\\)'", shell=True, capture_output=True, text=True).stdout)
print("mem:", subprocess.run("free -g | head -2", shell=True, capture_output=True, text=True).stdout)
print("nproc", os.cpu_count())
dev = torch.device("cuda:0")
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cuBLAS DGEMM n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s ({ms:.2f} ms)")
