#!/bin/bash
# One GPU round: smoke, tests, default bench (all legs), fp16/fp32 legs, the
# reference arm, ncu launch list of a bench step, ncu full captures of the
# chain, embed and boundary-IO kernels (+ raw/source CSV exports for profiles/).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --precision fp16 --steps 5 --no-converge > gpurun_out/bench_fp16.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --precision fp32 --steps 3 --iters 8 --no-converge > gpurun_out/bench_fp32.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>>gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --iters 4 --no-converge --no-extras > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2 -s 4 -c 1 -o gpurun_out/prof_chain -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_chain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_embed_tc -s 4 -c 1 -o gpurun_out/prof_embed -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_embed.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gather_phase|k_scatter_phase" -s 2 -c 2 -o gpurun_out/prof_io -f python tools/bench_io.py 1 > gpurun_out/ncu_io.log 2>&1
for r in prof_chain prof_embed prof_io; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>&1
done
ncu -i gpurun_out/prof_chain.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_chain_sass.csv 2>&1
ls -la gpurun_out | tail -30
