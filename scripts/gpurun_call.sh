cat > /tmp/st.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import synth
from paper_1904_12228_b200 import rsgrad as rs
dev = torch.device('cuda')
s = synth.stn_inputs(2, 16, 1024, 1024, cfg=2, device=dev)
y = rs.stn_fwd(s['x'], s['theta'])
dx, dt = rs.stn_bwd(s['x'], s['theta'], s['dy'])
torch.cuda.synchronize()
print("ok")
PY
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python /tmp/st.py 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -q -x -k "stn" > gpurun_out/pytest_stn.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_stn.log
python scripts/bench_layer.py 16 5 stn
