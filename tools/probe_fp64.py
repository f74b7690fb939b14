"""Probe: cuBLAS DGEMM / cuSOLVER DPOTRF fp64 rates on this B200 and host CPU facts.
Library numbers are context for the roofline denominator only (not product code)."""
import os, time, json, subprocess
import numpy as np
import torch

res = {}
res["nproc"] = os.cpu_count()
try:
    res["sched_affinity"] = len(os.sched_getaffinity(0))
except Exception:
    pass
res["cpu_model"] = subprocess.run("grep -m1 'model name' /proc/cpuinfo", shell=True, capture_output=True, text=True).stdout.strip()
res["mem"] = subprocess.run("free -g | head -2", shell=True, capture_output=True, text=True).stdout
d = torch.device("cuda:0")
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=d)
    b = torch.randn(n, n, dtype=torch.float64, device=d)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{n}_tflops_burst"] = 2 * n**3 / best / 1e9
    # sustained 4 s
    t0 = time.time(); cnt = 0
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        c = a @ b; cnt += 1
        if cnt % 4 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    res[f"dgemm_{n}_tflops_sustained"] = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
for m in (2048, 6197, 12288):
    x = torch.randn(m, m, dtype=torch.float64, device=d)
    h = x @ x.T / m + torch.eye(m, dtype=torch.float64, device=d) * 4
    for _ in range(2):
        torch.linalg.cholesky(h)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); L = torch.linalg.cholesky(h); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"cusolver_potrf_{m}_ms"] = best
    res[f"cusolver_potrf_{m}_tflops"] = m**3 / 3 / best / 1e9
# host BLAS
import scipy.linalg
for n in (2048,):
    a = np.random.rand(n, n); b = np.random.rand(n, n)
    t0 = time.perf_counter(); c = a @ b; t = time.perf_counter() - t0
    res["numpy_dgemm_2048_gflops"] = 2 * n**3 / t / 1e9
    t0 = time.perf_counter(); c = scipy.linalg.blas.dgemm(1.0, a, b); t = time.perf_counter() - t0
    res["scipy_dgemm_2048_gflops"] = 2 * n**3 / t / 1e9
print(json.dumps(res, indent=1))
