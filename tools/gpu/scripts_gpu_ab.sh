#!/bin/bash
# A/B of chain variants: parity tests under the variant, then bench chain timing.
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
for v in "$@"; do
  echo "=== $v"
  env $v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tensorcore or batch or fitted or full_size_sampled" > gpurun_out/ab_tests_${v//=/_}.log 2>&1; tail -2 gpurun_out/ab_tests_${v//=/_}.log
  for r in 1 2; do
    env $v timeout 180 python bench.py --steps 5 --warmup 3 --no-converge > gpurun_out/ab_${v//=/_}_$r.json 2>>gpurun_out/ab.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${v//=/_}_$r.json'));print('$v', round(d['value']/1e6,2), round(d['roofline']['chain_ms_per_launch'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  done
done
