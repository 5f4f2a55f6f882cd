python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_sensing.py tests/test_gpu_parity.py -q -x -k "width or gradients or stack or metrics or c_example" 2>&1 | tail -5
python - <<'PY'
import torch, numpy as np, synth, sys
sys.path.insert(0, '.')
from paper_1701_03891_b200 import DeepInverse
c = synth.CONFIGS["lowrate"]
phi = synth.make_phi(c.m, c.N, "bf16"); x = synth.make_images(c.n, 0, c.batch, c.n_blobs, c.n_rects)
y = synth.measure(phi, x, "bf16")
ctx = DeepInverse(phi, synth.make_params().rounded("bf16"), c.n, c.n, "bf16", max_batch=c.batch)
yd = torch.from_numpy(y).cuda().to(torch.bfloat16); xd = torch.from_numpy(x).cuda(); out = torch.empty((c.batch, c.n, c.n), device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for _ in range(3): ctx.recover_metrics(yd, xd, out); ctx.recover(yd, out); ctx.metrics(out, xd)
ts = []
for _ in range(10):
    ev[0].record(); ctx.recover_metrics(yd, xd, out); ev[1].record(); ctx.recover(yd, out); ctx.metrics(out, xd); ev[2].record(); torch.cuda.synchronize()
    ts.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
t = np.median(np.array(ts), axis=0)
print(f"fused recover+metrics {t[0]:.3f} ms, recover then metrics {t[1]:.3f} ms (incl. D2H of the metrics)")
PY
