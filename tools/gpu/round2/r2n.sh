python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_device_loop.py tests/test_gpu_delta.py -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
