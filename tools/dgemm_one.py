import torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2): c = a @ b
torch.cuda.synchronize()
# K1-like shape: (10112 x 656) x (656 x 654)
x = torch.randn(10112, 656, dtype=torch.float64, device="cuda"); k = torch.randn(656, 654, dtype=torch.float64, device="cuda")
for _ in range(3): y = x @ k
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): y = x @ k
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print("cublas K1-shape ms", ms, "TF", 2 * 10112 * 656 * 654 / ms / 1e9)
