"""Measure FMA-pipe peaks (FFMA, DFMA, FP64 DMMA) with the library's probes,
plus cuBLAS TF32/FP32/FP64 GEMM throughput for reference; writes JSON."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_05324_b200 import _lib

lib = _lib.load()
out = {}
for kind, name in ((0, "ffma"), (1, "dfma"), (2, "dmma_m8n8k4")):
    v = ctypes.c_double()
    lib.mt_peak_probe(kind, 40000, ctypes.byref(v))
    out[name + "_tflops"] = v.value

def gemm(dtype, tf32, n=8192, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype); b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3): a @ b
    torch.cuda.synchronize(); t = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): a @ b
    e1.record(); torch.cuda.synchronize()
    return 2 * n ** 3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12

out["cublas_tf32_tflops"] = gemm(torch.float32, True)
out["cublas_fp32_tflops"] = gemm(torch.float32, False)
out["cublas_fp64_tflops"] = gemm(torch.float64, False, n=4096, reps=5)
print(json.dumps(out))
