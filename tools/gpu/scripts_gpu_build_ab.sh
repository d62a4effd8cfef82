#!/bin/bash
# A/B of compile-time chain variants: for each MFP_NVCC_EXTRA value, rebuild,
# run the tensor-core parity tests, and two short benches (chain ms, frac).
mkdir -p gpurun_out
for v in "$@"; do
  echo "=== build [$v]"
  MFP_NVCC_EXTRA="$v" python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tensorcore or batch or fitted or full_size_sampled" > gpurun_out/abb_tests.log 2>&1; tail -1 gpurun_out/abb_tests.log
  for r in 1 2; do
    timeout 180 python bench.py --steps 5 --warmup 3 --no-converge > gpurun_out/abb.json 2>>gpurun_out/abb.err
    python -c "import json;d=json.load(open('gpurun_out/abb.json'));print('[$v]', round(d['value']/1e6,2), round(d['roofline']['chain_ms_per_launch'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  done
done
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
