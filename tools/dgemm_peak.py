"""cuBLAS DGEMM ceiling on the box (practical FP64 roofline reference) + tall-skinny shapes."""
import json, torch
def bench(m, n, k, reps=10):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"m": m, "n": n, "k": k, "ms": ms, "tflops": 2.0 * m * n * k / ms / 1e9}
out = [bench(8192, 8192, 8192), bench(16384, 16384, 16384, 3),
       bench(16384, 128, 16384), bench(16384, 256, 16384), bench(16384, 16384, 256), bench(98304, 512, 4096)]
for o in out: print(json.dumps(o))
print(torch.cuda.get_device_name(), torch.cuda.get_device_properties(0).total_memory / 2**30, "GiB")
