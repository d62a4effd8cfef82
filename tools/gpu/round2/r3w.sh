# session-3 measurement pass: default bench, fp16 leg, reference arm, launch list, ncu full captures of the d=128 chain and the embed
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], d["roofline"]["frac_vs_burst_peak"], "d256", d["roofline_d256"]["roofline"]["frac"], d["roofline_d256"]["value"], "fp16x", d["accuracy_mode_fp16x"]["value"], d["accuracy_mode_fp16x"]["chain_time_vs_headline_chain"], d["clocks"], d["boundary_io"]["gather"]["frac"], d["boundary_io"]["scatter"]["frac"])
print("ttc", json.dumps(d["time_to_converge"]["exact_subsolver"]))
print(json.dumps(d["roofline"]["iteration_breakdown_ms"]))
PY
timeout 600 python bench.py --precision fp16 --steps 5 --no-converge > gpurun_out/bench_fp16.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>>gpurun_out/bench.err
tail -c 300 gpurun_out/bench_fp16.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --iters 4 --no-converge --no-extras > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_chain_tc2$" -s 4 -c 1 -o gpurun_out/prof_chain -f python tools/d_probe.py 1 2 > gpurun_out/ncu_chain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_embed_tc -s 4 -c 1 -o gpurun_out/prof_embed -f python tools/d_probe.py 1 2 > gpurun_out/ncu_embed.log 2>&1
for r in prof_chain prof_embed; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_sass.csv 2>&1
done
ls -la gpurun_out | grep ncu-rep
