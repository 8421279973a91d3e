"""Per-bank timing of config 3 (dev): bank A TX (store), bank B TX (accumulate), both RX."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2008_00672_b200 import api, configs  # noqa: E402

mw = configs.config3()
plans = mw.plans()
mx = mw.mixed(plans)
S = 1024
grids = []
for i, (w, p) in enumerate(zip(mw.banks, plans)):
    g = torch.empty((S, w.B, p.row_active), dtype=torch.complex64, device="cuda")
    p.gen_qam(1 + i, 0, S, 6, g)
    grids.append(g)
wave = torch.zeros((S, mx.Q), dtype=torch.complex64, device="cuda")
outs = [torch.empty_like(g) for g in grids]
base = api._dev_ptr(wave)
st = torch.cuda.current_stream()


def timeit(f, n=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


(pA, oA), (pB, oB) = mx.banks
print("txA", timeit(lambda: pA.tx(grids[0], base + 8 * oA, S, wave_stride=mx.Q)))
print("txB acc", timeit(lambda: pB.tx(grids[1], base + 8 * oB, S, wave_stride=mx.Q, accumulate=True)))
print("txB store", timeit(lambda: pB.tx(grids[1], base + 8 * oB, S, wave_stride=mx.Q)))
print("rxA", timeit(lambda: pA.rx(base, mx.Q, oA + pA.useful0, outs[0], S, wave_stride=mx.Q)))
print("rxB", timeit(lambda: pB.rx(base, mx.Q, oB + pB.useful0, outs[1], S, wave_stride=mx.Q)))
