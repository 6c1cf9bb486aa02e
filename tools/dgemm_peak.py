"""cuBLAS DGEMM yardstick (torch.matmul float64): best of 10 at 8192^3 and sustained 4 s.

Builder tool, not product code: it gives the fp64 roofline denominator that
MEASURED_PEAKS.json does not carry.
"""
import json, time, subprocess, sys
import torch

def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(10):
        e0.record(); torch.matmul(a, b, out=c); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n**3 / (best * 1e-3) / 1e12
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader", "-lms", "200"], stdout=subprocess.PIPE, text=True)
    t0 = time.time(); cnt = 0
    e0.record()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b, out=c); cnt += 1
        if cnt % 4 == 0:
            torch.cuda.synchronize()
    e1.record(); e1.synchronize()
    sus = 2 * n**3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
    smi.terminate(); out = smi.communicate()[0].strip().splitlines()
    print(json.dumps({"dgemm_n": n, "fp64_tflops_burst": burst, "fp64_tflops_sustained": sus,
                      "clock_samples": out[-8:]}))

if __name__ == "__main__":
    main()
