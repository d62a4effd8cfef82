python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/d_probe.py 1 4 2>&1 | tail -2
