# final round-2 validation: smoke, full GPU suite, bench (all legs), launch list,
# memcheck of the changed lattice kernels (final lines, exact 8/4/2/1 per warp)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "d256", d["roofline_d256"]["roofline"]["frac"], d["roofline_d256"]["value"], "fp16x", d["accuracy_mode_fp16x"]["chain_time_vs_headline_chain"], d["clocks"], d["boundary_io"]["gather"]["frac"], d["boundary_io"]["scatter"]["frac"], d["time_to_converge"]["exact_subsolver"]["ms"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --iters 4 --no-converge --no-extras > /dev/null 2>&1
export MFP_NO_GRAPHS=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py tests/test_gpu_persistent.py -q -x -k "exact_fixed_k or exact_distributed_parity or persistent_bit_identical and not 4096" 2>&1 | tail -2
