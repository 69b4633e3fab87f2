# fp64 peak probe (measurement only): DFMA / DMMA issue rates and cuBLAS DGEMM via torch
./tools/fp64_probe
python - <<'PY'
import torch, time
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cublas dgemm n={n}: {2*n**3/ms/1e9:.2f} TFLOP/s")
m, k, n = 2500, 12700, 8192
a = torch.randn(m, k, dtype=torch.float64, device="cuda"); b = torch.randn(k, n, dtype=torch.float64, device="cuda")
for _ in range(3): a @ b
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): a @ b
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"cublas dgemm {m}x{k}x{n}: {2*m*n*k/ms/1e9:.2f} TFLOP/s  {ms:.2f} ms")
PY
