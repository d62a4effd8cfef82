python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
for np in 0 1 2; do for p in 1 2; do MFP_GELU_POLY=$np timeout 300 python tools/wfit_err.py $p; done; done > gpurun_out/wfit_err.txt 2>&1
cat gpurun_out/wfit_err.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; grep -E "^E .*assert|FAILED" gpurun_out/gpu_tests.log | head
for np in 0 1 2; do MFP_GELU_POLY=$np timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench_np$np.json 2>> gpurun_out/bench.err; done
MFP_GELU_POLY=1 timeout 600 python bench.py --no-converge --steps 5 --precision fp16 > gpurun_out/bench_fp16_np1.json 2>> gpurun_out/bench.err
for f in gpurun_out/bench_np*.json gpurun_out/bench_fp16_np1.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,2), d['roofline']['chain_ms_per_launch'])"; done
