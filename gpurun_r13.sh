cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/time_stages.py c2 20 >> gpurun_out/ab.log 2>&1
timeout 300 python - >> gpurun_out/ab.log 2>&1 <<'PY'
import sys, statistics
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2510_07514_b200 import hjcd, inputs
ch = inputs.panda(); rb = hjcd.Robot(ch)
th = torch.from_numpy(inputs.halton_configs(ch, 1000).astype(np.float32)).cuda()
tg = hjcd.fk(rb, th).contiguous()
for eps in ((1e-6, 1e-5), (1e-9, 1e-8)):
    c = hjcd.default_config(eps_p_fine=eps[0], eps_o_fine=eps[1])
    for _ in range(2): r = hjcd.solve_f64(rb, tg, c)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); r = hjcd.solve_f64(rb, tg, c); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    pe = r[1].cpu().numpy()
    print(f"solve_f64 eps {eps}: {statistics.median(ts):.3f} ms, status0 {(r[3] == 0).float().mean().item():.3f}, pos err p50 {np.median(pe):.2e} max {pe.max():.2e}")
PY
echo done
