# session-3 re-entry: full GPU suite + smoke + bench on the restored tree; ncu of the embed with source
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], d["roofline"]["frac_vs_burst_peak"], "d256", d["roofline_d256"]["roofline"]["frac"], d["roofline_d256"]["value"], "fp16x", d["accuracy_mode_fp16x"]["chain_time_vs_headline_chain"], d["clocks"], d["boundary_io"]["gather"]["frac"], d["boundary_io"]["scatter"]["frac"], d["gpu_launches"])
print(json.dumps(d["roofline"]["iteration_breakdown_ms"]))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_embed_tc -s 4 -c 1 -o gpurun_out/prof_embed -f python tools/d_probe.py 1 2 > gpurun_out/ncu_embed.log 2>&1
ncu -i gpurun_out/prof_embed.ncu-rep --page raw --csv > gpurun_out/prof_embed_raw.csv 2>&1
ncu -i gpurun_out/prof_embed.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_embed_sass.csv 2>&1
ncu -i gpurun_out/prof_embed.ncu-rep --page details --csv > gpurun_out/prof_embed_details.csv 2>&1
