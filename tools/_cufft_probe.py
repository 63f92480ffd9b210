"""Calibration: cuFFT (via torch.fft) on the C2 shapes -- cross-check only."""
import torch, time
def t(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)/n
for dt in (torch.float64, torch.float32):
    x = torch.randn(10000, 3584, dtype=dt, device="cuda")
    X = torch.fft.rfft(x, dim=1)
    Xt = X.t().contiguous()  # (1793, 10000) rho contiguous like our layout
    print(dt, "rfft rows (r2c) ms", round(t(lambda: torch.fft.rfft(x, dim=1)), 4))
    print(dt, "irfft rows (c2r) ms", round(t(lambda: torch.fft.irfft(X, n=3584, dim=1)), 4))
    print(dt, "fft along contiguous rho rows (1793 x 10000) ms", round(t(lambda: torch.fft.fft(Xt, dim=1)), 4))
    print(dt, "fft+ifft rho rows ms", round(t(lambda: torch.fft.ifft(torch.fft.fft(Xt, dim=1), dim=1)), 4))
    print(dt, "copy 287MB-equiv ms", round(t(lambda: x.clone()), 4))
