# (dropped variant) d = 128 chain head weights from the constant bank: spills, chain 0.1557 -> 0.1600 ms; full GPU suite + bench + timeline
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], d["roofline"]["frac_vs_burst_peak"], "d256", d["roofline_d256"]["roofline"]["frac"], d["roofline_d256"]["value"], "fp16x", d["accuracy_mode_fp16x"]["chain_time_vs_headline_chain"], d["clocks"], d["boundary_io"]["gather"]["frac"], d["boundary_io"]["scatter"]["frac"], d["gpu_launches"])
print(json.dumps(d["roofline"]["iteration_breakdown_ms"]))
PY
MFP_NVCC_EXTRA=-DMFP_TRACE python paper_2308_14258_b200/build.py --force > gpurun_out/build_trace.log 2>&1
timeout 300 python tools/chain_trace.py
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
