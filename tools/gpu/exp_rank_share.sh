python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary_io.py -q -x 2>&1 | tail -2
timeout 300 python tools/rank_share.py > gpurun_out/rank_share.json 2> gpurun_out/rank_share.err; cut -c1-250 gpurun_out/rank_share.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-converge --no-extras
