# session-3 final measurement pass: smoke, full GPU suite, default bench + fp16/fp32/reference legs, launch list,
# ncu full captures of the d=128 / d=256 / FP16X chains and the embed, rank shares at d = 128 / 256
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], d["roofline"]["frac_vs_burst_peak"], "d256", d["roofline_d256"]["roofline"]["frac"], d["roofline_d256"]["value"], "fp16x", d["accuracy_mode_fp16x"]["value"], d["accuracy_mode_fp16x"]["chain_time_vs_headline_chain"], d["clocks"], d["boundary_io"]["gather"]["frac"], d["boundary_io"]["scatter"]["frac"])
print(json.dumps(d["roofline"]["iteration_breakdown_ms"]))
print(json.dumps(d["time_to_converge"]))
PY
timeout 600 python bench.py --precision fp16 --steps 5 --no-converge > gpurun_out/bench_fp16.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --precision fp32 --steps 3 --iters 8 --no-converge > gpurun_out/bench_fp32.json 2>>gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>>gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --iters 4 --no-converge --no-extras > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_chain_tc2$" -s 4 -c 1 -o gpurun_out/prof_chain -f python tools/d_probe.py 1 2 > gpurun_out/ncu_chain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2w -s 4 -c 1 -o gpurun_out/prof_chain256 -f python tools/d_probe.py 1 2 > gpurun_out/ncu_chain256.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2s -s 4 -c 1 -o gpurun_out/prof_chain_fp16x -f python tools/d_probe.py 3 2 > gpurun_out/ncu_chain_fp16x.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_embed_tc -s 4 -c 1 -o gpurun_out/prof_embed -f python tools/d_probe.py 1 2 > gpurun_out/ncu_embed.log 2>&1
for s in "4096 4096" "2048 4096" "2048 2048" "1024 2048"; do timeout 120 python tools/share_probe.py $s 1 2>&1 | grep ms; MFP_PROBE_D=256 timeout 120 python tools/share_probe.py $s 1 2>&1 | grep ms; done > gpurun_out/rank_share.txt
cat gpurun_out/rank_share.txt
ls gpurun_out/*.ncu-rep
