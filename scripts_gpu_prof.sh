#!/bin/bash
# Full ncu captures of the chain and embed kernels (one launch each, C5 phase).
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc -s 4 -c 1 -o gpurun_out/prof_chain -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_embed -s 4 -c 1 -o gpurun_out/prof_embed -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
