python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; grep -E "^E .*assert|FAILED" gpurun_out/gpu_tests.log | head
timeout 600 python bench.py --no-converge > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --no-converge --precision fp16 --steps 5 > gpurun_out/bench_fp16.json 2>> gpurun_out/bench.err; cat gpurun_out/bench_fp16.json
