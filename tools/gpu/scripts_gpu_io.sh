#!/bin/bash
# boundary-IO kernels: GPU tests, timing leg, ncu DRAM bytes of one launch each.
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_boundary_io.py -q -x > gpurun_out/io_tests.log 2>&1; tail -15 gpurun_out/io_tests.log
timeout 300 python tools/bench_io.py 10 noflush > gpurun_out/bench_io.json 2> gpurun_out/bench_io.err; cat gpurun_out/bench_io.json; tail -3 gpurun_out/bench_io.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scatter_phase" -s 1 -c 1 -o gpurun_out/prof_io -f python tools/bench_io.py 1 > gpurun_out/ncu_io.log 2>&1
ncu -i gpurun_out/prof_io.ncu-rep --page raw --csv > gpurun_out/prof_io_raw.csv 2>&1

