"""CPU checks of bench.py's driver contract that need no GPU: the reference arm
(the fp64 oracle on the host cores) prints one well-formed JSON line, and the
strong / weak scaling domains follow SURVEY §8(d)."""
import json
import os
import subprocess
import sys

from tests.conftest import ROOT

sys.path.insert(0, ROOT)


def test_scaling_domains():
    import bench
    assert [bench.domain(n, "strong") for n in (1, 2, 4, 8)] == [(4096, 4096)] * 4
    assert [bench.domain(n, "weak") for n in (1, 2, 4, 8)] == [(1024, 2048), (2048, 2048), (2048, 4096),
                                                                 (4096, 4096)]
    assert bench.preds_per_iter(4096, 4096) == 65025 == bench.PRED_PER_ITER


def test_reference_arm_json_line():
    env = dict(os.environ, OMP_NUM_THREADS="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"].startswith("C5")
