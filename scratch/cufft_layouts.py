"""cuFFT timings for the 2048^2 x 32 inverse FFT2 split by axis (layout study)."""
import torch
def t(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
B, Y, X = 32, 2048, 2048
g = torch.randn(B, Y, X, dtype=torch.complex64, device="cuda")
print("ifft2 [b][y][x]        %.3f ms" % t(lambda: torch.fft.ifft2(g, out=g)))
h = torch.randn(Y, B * X, dtype=torch.complex64, device="cuda")
print("ifft dim0 [y][b*x]     %.3f ms" % t(lambda: torch.fft.ifft(h, dim=0, out=h)))
r = torch.randn(Y * B, X, dtype=torch.complex64, device="cuda")
print("ifft rows [y*b][x]     %.3f ms" % t(lambda: torch.fft.ifft(r, dim=1, out=r)))
print("ifft dim1 [b][y][x]    %.3f ms" % t(lambda: torch.fft.ifft(g, dim=1, out=g)))
