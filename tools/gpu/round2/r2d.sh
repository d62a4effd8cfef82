mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_d256.py -x -q > gpurun_out/d256_tests.log 2>&1
tail -30 gpurun_out/d256_tests.log
timeout 300 python tools/d_probe.py 1 4 > gpurun_out/d_probe.jsonl 2>&1; cat gpurun_out/d_probe.jsonl
