"""cuBLAS DGEMM launch configuration probe (builder tool; run under ncu)."""
import torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    c = a @ b
# the trailing-update shape: (32768 x 128) @ (128 x 32640)
y = torch.randn(32768, 128, dtype=torch.float64, device="cuda")
w = torch.randn(128, 32640, dtype=torch.float64, device="cuda")
c2 = torch.empty(32768, 32640, dtype=torch.float64, device="cuda")
torch.addmm(c2, y, w, out=c2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); torch.addmm(c2, y, w, out=c2); e1.record(); e1.synchronize()
print("cuBLAS rank-128 update 32768x32640: %.2f TFLOP/s" % (2 * 32768 * 32640 * 128 / e0.elapsed_time(e1) / 1e9))
yt = torch.randn(128, 32768, dtype=torch.float64, device="cuda")
e0.record(); r = yt @ c2[:, :32640]; e1.record(); e1.synchronize()
print("cuBLAS Y^T C 128x32640 K=32768: %.2f TFLOP/s" % (2 * 32768 * 32640 * 128 / e0.elapsed_time(e1) / 1e9))
