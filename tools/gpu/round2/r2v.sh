python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 300 python tools/d_probe.py 1 4 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_p2p_put.py tests/test_gpu_p2p.py -q -x 2>&1 | tail -2
