timeout 900 python -m pytest tests -m gpu -q -x -k "bicubic or variants" > gpurun_out/pytest_f3.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_f3.log
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import synth
from paper_1904_12228_b200 import rsgrad as rs
dev = torch.device('cuda')
si = synth.stn_inputs(4, 16, 512, 512, cfg=2, device=dev)
dx, dt = torch.empty_like(si['x']), torch.empty_like(si['theta'])
def t(fn, r=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(r): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / r * 1e3
print('auto both', t(lambda: rs.stn_bicubic_bwd(si['x'], si['theta'], si['dy'], out=(dx, dt))))
print('gather both', t(lambda: rs.stn_bicubic_bwd(si['x'], si['theta'], si['dy'], algo='gather', out=(dx, dt))))
print('dtheta only', t(lambda: rs.stn_bicubic_bwd(si['x'], si['theta'], si['dy'], need_dx=False, out=(None, dt))))
print('dx atomic only', t(lambda: rs.stn_bicubic_bwd(si['x'], si['theta'], si['dy'], algo='scatter_atomic', need_dtheta=False, out=(dx, None))))
PY
