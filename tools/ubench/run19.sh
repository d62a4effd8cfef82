python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log; grep -E "^E .*assert|FAILED|Error" gpurun_out/gpu_tests.log | head -5
MFP_CHAIN_VARIANT=3 timeout 900 python -m pytest tests -m gpu -q -x -k "tensorcore or batch or fitted" > gpurun_out/gpu_tests3.log 2>&1; tail -1 gpurun_out/gpu_tests3.log
timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench.json 2>> gpurun_out/bench.err
MFP_CHAIN_VARIANT=3 timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench3.json 2>> gpurun_out/bench.err
MFP_L0_MMA=1 timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench_l0.json 2>> gpurun_out/bench.err
for f in gpurun_out/bench.json gpurun_out/bench3.json gpurun_out/bench_l0.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,2), d['roofline']['chain_ms_per_launch'])"; done
