mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fp16x.py tests/test_gpu_bench_parity.py -q -s > gpurun_out/fp16x_tests.log 2>&1
grep -E "FP16X|C5 prec|interior|passed|failed|Error" gpurun_out/fp16x_tests.log | tail -40
timeout 300 python tools/d_probe.py 3 4 > gpurun_out/d_probe3.jsonl 2>&1; cat gpurun_out/d_probe3.jsonl
