python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests/test_gpu_sensing.py -q -x -k metrics 2>&1 | tail -2
for w in 1,64,64,32,1 1,64,128,32,1 1,64,128,128,32,1 1,32,128,64,32,1; do timeout 300 python tools/time_stack.py bf16 4096 64 410 $w; done
timeout 300 python tools/time_stack.py f32 256 64 410 1,64,128,32,1
python - <<'PY'
import torch, numpy as np, synth, sys, json, time
sys.path.insert(0, '.')
from paper_1701_03891_b200 import DeepInverse
from tests.test_gpu_stack import stack_params
for prec, widths in [("bf16", (1, 64, 128, 64, 32, 1)), ("bf16", (1, 64, 32, 1)), ("f32", (1, 64, 128, 32, 1))]:
    B, n = 256, 64
    p = stack_params(widths).rounded("bf16" if prec == "bf16" else "f32")
    phi = synth.make_phi(410, n * n, "bf16" if prec == "bf16" else "f32")
    x = synth.make_images(n, 0, B, 8, 4); y = synth.measure(phi, x, "bf16" if prec == "bf16" else "f32")
    ctx = DeepInverse(phi, p, n, n, prec, max_batch=B)
    yd = torch.from_numpy(y).cuda().to(ctx.storage_dtype); xd = torch.from_numpy(x).cuda()
    for _ in range(2): loss, g = ctx.train_grad(yd, xd); ctx.sgd_step(g, 1e-6, 0.9)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): loss, g = ctx.train_grad(yd, xd); ctx.sgd_step(g, 1e-6, 0.9)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    print(json.dumps({"train": prec, "widths": widths, "batch": B, "ms_per_step": round(dt * 1e3, 2), "images_per_s": round(B / dt)}))
PY
