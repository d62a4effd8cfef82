#!/bin/bash
# One GPU round: smoke, tests, default bench (all legs), fp16/fp32 legs, ncu
# launch list, ncu full captures of the chain and embed kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --precision fp16 --steps 5 --no-converge > gpurun_out/bench_fp16.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --precision fp32 --steps 3 --iters 8 --no-converge > gpurun_out/bench_fp32.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>>gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --iters 4 --no-converge > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2 -s 4 -c 1 -o gpurun_out/prof_chain -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_chain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_embed_tc -s 4 -c 1 -o gpurun_out/prof_embed -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_embed.log 2>&1
ls -la gpurun_out | tail -30
