# after the exact-path changes: smoke, full GPU suite, default bench
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "d256", d["roofline_d256"]["roofline"]["frac"], "fp16x", d["accuracy_mode_fp16x"]["chain_time_vs_headline_chain"], d["clocks"], d["boundary_io"]["gather"]["frac"], d["boundary_io"]["scatter"]["frac"])
print("ttc exact", d["time_to_converge"]["exact_subsolver"]["ms"], "fit C5", d["time_to_converge"]["sdnet_w_fit_mae_0.05_bench_domain"]["ms"])
PY
