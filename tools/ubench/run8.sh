python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log; grep -E "^E .*assert|FAILED|Error" gpurun_out/gpu_tests.log | head -5
timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench.json 2>> gpurun_out/bench.err
MFP_L0_SIMT=1 timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench_l0simt.json 2>> gpurun_out/bench.err
for f in gpurun_out/bench.json gpurun_out/bench_l0simt.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,2), d['roofline']['chain_ms_per_launch'])"; done
