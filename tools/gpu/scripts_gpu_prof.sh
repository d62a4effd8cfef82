#!/bin/bash
# ncu --set full of the chain kernel (one C5 phase launch) + source-level stall export.
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2 -s 4 -c 1 -o gpurun_out/prof_chain -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_chain.log 2>&1
ncu -i gpurun_out/prof_chain.ncu-rep --page raw --csv > gpurun_out/prof_chain_raw.csv 2>&1
ncu -i gpurun_out/prof_chain.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_chain_sass.csv 2>&1
ncu -i gpurun_out/prof_chain.ncu-rep --page details --csv > gpurun_out/prof_chain_details.csv 2>&1
ls -la gpurun_out
