python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_nccl1.py -q 2>&1 | tail -4
