mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
tail -8 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['roofline']['iteration_breakdown_ms'])"
