"""Context numbers on the box: cuBLAS DGEMM and cuSOLVER batched Cholesky (library, not product)."""
import torch, time
d = torch.device("cuda:0")
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=d)
    b = torch.randn(n, n, dtype=torch.float64, device=d)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"DGEMM n={n}: {ms:.2f} ms {2*n**3/ms/1e9:.1f} TFLOP/s")
for n, B in ((4096, 8), (2048, 32)):
    x = torch.randn(B, n, n, dtype=torch.float64, device=d)
    A = x @ x.transpose(1, 2) + n * torch.eye(n, dtype=torch.float64, device=d)
    for _ in range(2):
        L = torch.linalg.cholesky(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L = torch.linalg.cholesky(A)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"cusolver cholesky n={n} B={B}: {ms:.2f} ms  {B*n**3/3/ms/1e9:.2f} TFLOP/s  {B/ms*1e3:.1f} fact/s")
