mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sine.py -q -s > gpurun_out/sine_tests.log 2>&1; grep -E "MAE|passed|failed" gpurun_out/sine_tests.log
timeout 900 python tools/e6_batching.py > gpurun_out/e6.json 2> gpurun_out/e6.err; cat gpurun_out/e6.err | tail -9
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --iters 4 --no-converge --no-extras > gpurun_out/ncu_launch_bench.log 2>&1
tail -2 gpurun_out/ncu_launch_bench.log
