python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; grep -E "^E .*assert|FAILED" gpurun_out/gpu_tests.log | head
timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench.json 2>> gpurun_out/bench.err
timeout 600 python bench.py --no-converge --steps 5 --precision fp16 > gpurun_out/bench_fp16.json 2>> gpurun_out/bench.err
for f in gpurun_out/bench.json gpurun_out/bench_fp16.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,2), d['roofline']['chain_ms_per_launch'])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2 -s 4 -c 1 -o gpurun_out/prof_chain4 -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_chain.log 2>&1; tail -1 gpurun_out/ncu_chain.log
