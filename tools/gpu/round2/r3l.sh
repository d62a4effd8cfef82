python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_d256.py -q -k fewer 2>&1 | tail -4
