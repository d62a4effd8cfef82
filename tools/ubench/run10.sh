MFP_NVCC_EXTRA="-DMFP_OOO_ISSUE" python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "tensorcore or batch" > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench_ooo.json 2>> gpurun_out/bench.err
MFP_NVCC_EXTRA="-DMFP_OOO_ISSUE -DMFP_TRACE" python paper_2308_14258_b200/build.py --force >> gpurun_out/build.log 2>&1
timeout 300 python tools/chain_trace.py > gpurun_out/trace_ooo.txt 2>&1; head -12 gpurun_out/trace_ooo.txt
python paper_2308_14258_b200/build.py --force >> gpurun_out/build.log 2>&1
timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench.json 2>> gpurun_out/bench.err
for f in gpurun_out/bench.json gpurun_out/bench_ooo.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,2), d['roofline']['chain_ms_per_launch'])"; done
