set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes tools/ubench/pipes.cu && /tmp/pipes > gpurun_out/pipes.txt 2>&1
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-converge > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
MFP_EMBED_SIMT=1 timeout 600 python bench.py --no-converge --steps 5 > gpurun_out/bench_simt.json 2>> gpurun_out/bench.err; cat gpurun_out/bench_simt.json
cat gpurun_out/pipes.txt
