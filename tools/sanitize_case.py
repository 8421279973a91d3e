"""One small TX + fused/direct RX of a BASELINE config through the C ABI, for
compute-sanitizer (tools/sanitize.sh): python tools/sanitize_case.py CONFIG UNITS [SYMBOLS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2008_00672_b200 import configs  # noqa: E402

name, units = sys.argv[1], int(sys.argv[2])
w = configs.get(name)
if len(sys.argv) > 3 and hasattr(w, "cp"):
    w.cp = w.cp[:int(sys.argv[3])]
if hasattr(w, "banks"):
    plans = w.plans()
    mx = w.mixed(plans)
    grids = []
    for i, (b, p) in enumerate(zip(w.banks, plans)):
        g = torch.empty((units, b.B, p.row_active), dtype=torch.complex64, device="cuda")
        p.gen_qam(1 + i, 0, units, w.bits_per_symbol, g)
        grids.append(g)
    wave = torch.empty((units, mx.Q), dtype=torch.complex64, device="cuda")
    mx.tx(grids, wave, units)
    outs = [torch.empty_like(g) for g in grids]
    mx.rx(wave, outs, units, fused=True)
else:
    p = w.plan()
    g = torch.empty((units, w.B, p.row_active), dtype=torch.complex64, device="cuda")
    p.gen_qam(1, 0, units, w.bits_per_symbol, g)
    wave = torch.empty((units, p.Q), dtype=torch.complex64, device="cuda")
    p.tx(g, wave, units)
    out = torch.empty_like(g)
    for fused in (True, False):
        p.rx(wave, p.Q, p.useful0, out, units, fused=fused)
torch.cuda.synchronize()
print("ok", name, units, os.environ.get("FCW_CHUNK", "-"))
