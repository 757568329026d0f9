"""FP64 / complex128 dense throughput of this GPU (cuBLAS DGEMM / ZGEMM through torch):
the denominator for the setup factorisation's FP64 fraction (MEASURED_PEAKS.json has none)."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
out = {}
for name, dt, n, fl in (("dgemm", torch.float64, 8192, 2), ("zgemm", torch.complex128, 4096, 8)):
    a = torch.randn(n, n, dtype=dt, device="cuda"); b = torch.randn(n, n, dtype=dt, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    out[name + "_tflops"] = fl * n ** 3 / (best / 1e3) / 1e12
print(json.dumps(out))
