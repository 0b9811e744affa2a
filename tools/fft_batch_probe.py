"""cuFFT (through torch.fft) time per signal for config 4's length-L c128 FFT vs batch size (tools only)."""
import torch
L = 737280
for B in (1, 2, 4, 8, 16):
    x = torch.randn(B, L, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        torch.fft.fft(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.fft.fft(x)
    e1.record()
    torch.cuda.synchronize()
    print(f"batch {B}: {e0.elapsed_time(e1) / 10 / B * 1000:.1f} us per signal", flush=True)
