"""Probe FP64 peaks on the B200 box: cuBLAS DGEMM (torch.matmul fp64), a DMMA / DFMA
microbenchmark compiled here, and a read-only HBM stream. Writes gpurun_out/peaks_fp64.json.
Scratch measurement tool (not product code)."""
import json, os, subprocess, sys, time, ctypes
import torch

out = {}
dev = torch.device("cuda:0")
torch.cuda.synchronize()
def timeit(fn, reps=10):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best
for n in (4096, 8192, 10000):
    a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
    t = timeit(lambda: torch.matmul(a, b), reps=5)
    out[f"cublas_dgemm_{n}_tflops"] = 2 * n**3 / t / 1e12
# tall-skinny E.X via cuBLAS at n=10000
n = 10000
E = torch.randn(n, n, dtype=torch.float64, device=dev)
for k in (16, 32, 64, 96, 128):
    X = torch.randn(n, k, dtype=torch.float64, device=dev)
    t = timeit(lambda: torch.matmul(E, X), reps=10)
    out[f"cublas_EX_n{n}_k{k}_us"] = t * 1e6
    out[f"cublas_EX_n{n}_k{k}_GBs"] = 8 * n * n / t / 1e9
# read-only stream: sum of 1 GiB fp64
x = torch.ones(2**27, dtype=torch.float64, device=dev)
t = timeit(lambda: x.sum(), reps=10)
out["torch_sum_read_GBs"] = 8 * 2**27 / t / 1e9
y = torch.empty_like(x)
t = timeit(lambda: y.copy_(x), reps=10)
out["torch_copy_GBs"] = 16 * 2**27 / t / 1e9
# microbench
so = sys.argv[1] if len(sys.argv) > 1 else None
if so and os.path.exists(so):
    lib = ctypes.CDLL(so)
    lib.probe_dmma.restype = ctypes.c_double
    lib.probe_dfma.restype = ctypes.c_double
    out["dmma_tflops"] = lib.probe_dmma()
    out["dfma_tflops"] = lib.probe_dfma()
out["device"] = torch.cuda.get_device_name(0)
out["sm_count"] = torch.cuda.get_device_properties(0).multi_processor_count
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/peaks_fp64.json", "w"), indent=1)
