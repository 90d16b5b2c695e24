"""Check ofdmr_periodogram (1024 x 256) of the library named by OFDMR_LIB against a torch.fft fp32
restatement on random frames (a development check for kernel variants; the parity tests compare
against the oracle).  Prints the worst per-frame max|dP| / max(P)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_03883_b200.receiver import Receiver  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 300
for win in ("rectangular", "hamming"):
    g = torch.Generator(device="cuda").manual_seed(7)
    h = torch.randn(F, 1024, 256, dtype=torch.complex64, device="cuda", generator=g)
    p = torch.empty(F, 1024, 256, dtype=torch.float32, device="cuda")
    rx = Receiver(1024, 256, window=win)
    rx._stream()
    rx._lib.ofdmr_periodogram(rx._h, h.data_ptr(), p.data_ptr(), F)
    torch.cuda.synchronize()
    n = torch.arange(1024, device="cuda", dtype=torch.float64)
    m = torch.arange(256, device="cuda", dtype=torch.float64)
    if win == "hamming":
        wk = (0.54 - 0.46 * torch.cos(2 * torch.pi * n / 1023)).float()
        wl = (0.54 - 0.46 * torch.cos(2 * torch.pi * m / 255)).float()
    else:
        wk = torch.ones(1024, device="cuda")
        wl = torch.ones(256, device="cuda")
    worst = 0.0
    for f0 in range(0, F, 50):
        x = h[f0:f0 + 50] * (wk[:, None] * wl[None, :])
        X = torch.fft.fft(torch.fft.ifft(x, dim=1, norm="forward"), dim=2)
        pr = torch.fft.fftshift((X.abs() ** 2) / (1024 * 256), dim=2)
        d = (p[f0:f0 + 50] - pr).abs().amax(dim=(1, 2)) / pr.amax(dim=(1, 2))
        worst = max(worst, float(d.max()))
    print(f"{os.path.basename(os.environ.get('OFDMR_LIB', 'default'))} {win}: worst rel err {worst:.2e}",
          "OK" if worst < 1e-5 else "FAIL")
