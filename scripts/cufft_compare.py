"""cuFFT timed beside the library's own FFT passes (comparison only: north_star (c) asks for it;
nothing in the product calls cuFFT).  For the transform sizes of the bench configs it times
  * cuFFT Z2Z through torch.fft.fft (out-of-place, complex128),
  * the library's standalone FFT entry point nfft45_dft (the four-step Stockham passes the plan build
    and the forward NFFTs use),
with CUDA events on one stream, inputs larger than L2 for the batched sizes, and checks that both
agree to roundoff.  The solve chains never run a standalone FFT: their passes are fused with the
band / deconvolution / kernel-sample stages, so the table also lists, for C4, what
the two HBM passes of one FFT_2P cost inside the chain (bench.py's kernel table: bm_col + bm_row).
usage: python scripts/cufft_compare.py [out.md]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1604_06236_b200 as nf
from paper_1604_06236_b200 import _device, _lib

dev = 0
torch.cuda.set_device(dev)
SIZES = [(1 << 17, 1024, "C4 FFT_2P"), (1 << 16, 1024, "C4 FFT_P"), (1 << 21, 1, "C3 FFT_2P"), (1 << 20, 1, "C3 FFT_P"),
         (1 << 19, 1, "C5 FFT_2P"), (1 << 18, 1, "C5 FFT_P"), (8192, 64, "C2 FFT_2P"), (4096, 64, "C2 FFT_P")]


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rows = []
g = torch.Generator(device=f"cuda:{dev}")
g.manual_seed(1604)
for n, batch, label in SIZES:
    x = torch.complex(torch.randn(batch, n, generator=g, device=f"cuda:{dev}", dtype=torch.float64),
                      torch.randn(batch, n, generator=g, device=f"cuda:{dev}", dtype=torch.float64))
    y_cu = torch.empty_like(x)
    y_me = torch.empty_like(x)
    st = _device.stream_handle(dev)
    reps = 10 if batch > 1 and n >= (1 << 16) else 50
    ms_cu = timed(lambda: torch.fft.fft(x, out=y_cu), reps)
    ms_me = timed(lambda: _lib.call("nfft45_dft", x.data_ptr(), y_me.data_ptr(), batch, n, -1, st), reps)
    err = float((y_me - y_cu).abs().max() / y_cu.abs().max())
    gb = 32.0 * n * batch / 1e9  # algorithmic bytes: read + write one complex128 per point
    rows.append((label, n, batch, ms_cu, gb / ms_cu * 1e3, ms_me, gb / ms_me * 1e3, err))
    del x, y_cu, y_me

lines = ["| transform | N | batch | cuFFT ms | cuFFT GB/s (32 B/pt) | nfft45_dft ms | nfft45_dft GB/s | max diff / max |",
         "|---|---|---|---|---|---|---|---|"]
for r in rows:
    lines.append("| %s | %d | %d | %.4f | %.0f | %.4f | %.0f | %.1e |" % r)
out = "\n".join(lines)
print(out)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        f.write(out + "\n")
