python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "communication or chunked or distributed" 2>&1 | tail -3
timeout 900 python tools/iters_to_mae.py --only "exact fp32" --grids 1x1,2x4 --exchange-every 1,2,4,8 --chunk 40 > gpurun_out/iters_ca.json 2> gpurun_out/iters_ca.err; cut -c1-200 gpurun_out/iters_ca.err
