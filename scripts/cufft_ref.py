"""Time cuFFT (library) on the C2 row-convolution shape for comparison with
the hand-written passes: 65536 real fibres of 256, circulant embedding 512."""
import torch
torch.backends.cuda.cufft_plan_cache.max_size = 16
dev = "cuda"
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
x = torch.randn(65536, 256, dtype=torch.float64, device=dev)
sym = torch.randn(257, dtype=torch.float64, device=dev)
def conv_r2c():
    X = torch.fft.rfft(x, n=512, dim=1)
    X *= sym
    return torch.fft.irfft(X, n=512, dim=1)[:, :256]
z = torch.randn(32768, 512, dtype=torch.complex128, device=dev)
symc = torch.randn(512, dtype=torch.complex128, device=dev)
def conv_c2c():
    Z = torch.fft.fft(z, dim=1)
    Z *= symc
    return torch.fft.ifft(Z, dim=1)
print(f"cuFFT rfft/irfft conv (65536x256 -> 512): {t(conv_r2c):.1f} us")
print(f"cuFFT c2c fft/ifft 512 (32768 lanes): {t(conv_c2c):.1f} us")
y = torch.randn(65536, 512, dtype=torch.float64, device=dev)
print(f"cuFFT rfft only 512 (65536): {t(lambda: torch.fft.rfft(y, dim=1)):.1f} us")
print(f"cuFFT c2c fft only 512 (32768): {t(lambda: torch.fft.fft(z, dim=1)):.1f} us")
zz = torch.randn(65536, 256, dtype=torch.complex128, device=dev)
print(f"cuFFT c2c fft only 256 (65536): {t(lambda: torch.fft.fft(zz, dim=1)):.1f} us")
