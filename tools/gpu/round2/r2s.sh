python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_p2p_put.py tests/test_gpu_p2p.py -q -x 2>&1 | tail -15
