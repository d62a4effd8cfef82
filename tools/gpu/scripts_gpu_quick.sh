#!/bin/bash
# Quick GPU round: parity tests, bench, ncu capture of the chain kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --precision fp16 --steps 3 --no-converge > gpurun_out/bench_fp16.json 2>>gpurun_out/bench.err; cat gpurun_out/bench_fp16.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc -s 4 -c 1 -o gpurun_out/prof_chain -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_chain.log 2>&1
