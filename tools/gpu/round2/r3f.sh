python paper_2308_14258_b200/build.py > /dev/null 2>&1
for v in 0 8 4 2 1; do MFP_EXACT_SUB=$v timeout 300 python - <<'PY'
import os, sys, json
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2308_14258_b200 as mfp
from mfp_inputs import gp_boundary
out = {"MFP_EXACT_SUB": os.environ.get("MFP_EXACT_SUB")}
for nx, ny in ((4096, 4096), (2048, 4096), (2048, 2048), (1024, 2048)):
    cfg = mfp.make_config(nx, ny, subsolver=mfp.EXACT_LAPLACE, check_every=16)
    m = mfp.Mfp(cfg, mfp.make_net(), None)
    g = torch.from_numpy(gp_boundary(nx, ny, 0)).cuda()
    u = torch.empty((ny + 1, nx + 1), device="cuda")
    m.solve_device(g, 64, 0.0, u); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(m.stream); m.solve_device(None, 1024, 0.0, None); e1.record(m.stream); e1.synchronize()
    out[f"{nx}x{ny}_us_per_iteration"] = 1000 * e0.elapsed_time(e1) / 1024
    out[f"{nx}x{ny}_usum"] = float(u.double().sum())
print(json.dumps(out))
PY
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_persistent.py tests/test_gpu_delta.py -q -k "exact or persist or delta" 2>&1 | tail -1
