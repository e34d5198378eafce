"""Library reference point: cuBLASLt int8 GEMM (torch._int_mm, int8 x int8 -> int32) on this box."""
import json
import torch

res = {}
for n in (4096, 8192, 16384):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()   # column-major B (TN)
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10 if n <= 8192 else 4
    e0.record()
    for _ in range(reps):
        torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[f"int_mm_{n}_tops"] = round(2 * n ** 3 / (ms * 1e-3) / 1e12, 1)
    a16 = a.to(torch.bfloat16)
    b16 = b.to(torch.bfloat16)
    torch.matmul(a16, b16)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        torch.matmul(a16, b16)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[f"bf16_mm_{n}_tflops"] = round(2 * n ** 3 / (ms * 1e-3) / 1e12, 1)
print(json.dumps(res))
