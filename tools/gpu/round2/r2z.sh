python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "exact" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_device_loop.py tests/test_gpu_delta.py -q -x 2>&1 | tail -3
for v in 1 0; do MFP_NO_PERSIST=$v timeout 300 python - <<'PY'
import os, sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2308_14258_b200 as mfp
from mfp_inputs import gp_boundary
nx = ny = 4096
cfg = mfp.make_config(nx, ny, subsolver=mfp.EXACT_LAPLACE, check_every=16)
m = mfp.Mfp(cfg, mfp.make_net(), None)
g = torch.from_numpy(gp_boundary(nx, ny, 0)).cuda()
u = torch.empty((ny + 1, nx + 1), device="cuda")
m.solve_device(g, 64, 0.0, u)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(m.stream); rep = m.solve_device(g, 512, 0.0, u); e1.record(m.stream); e1.synchronize()
u1 = u.clone()
tol = 1e-6 * float(np.max(np.abs(gp_boundary(nx, ny, 0))))
e0.record(m.stream); rc = m.solve_device(g, 200000, tol, u); e1.record(m.stream); e1.synchronize()
print(json.dumps({"persist_disabled": os.environ.get("MFP_NO_PERSIST"), "ms_per_iter_512": None,
                  "ttc_ms": e0.elapsed_time(e1), "iters": rc.iterations, "u_sum": float(u1.double().sum())}))
PY
done
