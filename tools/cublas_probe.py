"""cuBLAS (torch.matmul, bf16) on the LAS-R101 stage-3 GEMM shapes, for context on
what a library GEMM reaches at these skinny shapes (not a product path)."""
import torch

shapes = {"conv1 (M=50176,K=1024,N=256)": (50176, 1024, 256),
          "conv2 r=.5 (M=25088,K=2304,N=256)": (25088, 2304, 256),
          "conv3 r=.5 (M=25088,K=256,N=1024)": (25088, 256, 1024),
          "stage2 conv1 (M=200704,K=512,N=128)": (200704, 512, 128),
          "stage0 conv1 (M=802816,K=256,N=64)": (802816, 256, 64)}
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for name, (m, k, n) in shapes.items():
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ b
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    t = sorted(ts)[len(ts) // 2]
    byt = (m * k + k * n + m * n) * 2
    print(f"{name}: {t:.1f} us  {2 * m * n * k / t / 1e6:.0f} TF/s  {byt / t / 1e3:.0f} GB/s")
