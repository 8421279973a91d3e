for env in "X=1" "X=2" "FCW_CHUNK_TX=4" "FCW_CHUNK_TX=4" "FCW_CHUNK_TX=8" "FCW_CHUNK_TX=16"; do
  env $env python bench.py --config c4 --no-cpu --no-e2e --steps 5 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', d['kernels_ms'])"
done
python - <<'PY'
import torch, time
from paper_2008_00672_b200 import configs
w = configs.config4(); p = w.plan()
S = 4
g = torch.empty((S, w.B, p.row_active), dtype=torch.complex64, device="cuda"); p.gen_qam(1, 0, S, 8, g)
wave = torch.empty((S, p.Q), dtype=torch.complex64, device="cuda")
for i in range(6):
    torch.cuda.synchronize(); t = time.perf_counter(); p.tx(g, wave, S); torch.cuda.synchronize(); print("tx", i, round((time.perf_counter()-t)*1e3, 3), "ms", float(wave.abs().max()))
PY
