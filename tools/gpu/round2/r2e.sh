# round-2 measurement pass: bench (all legs), launch list, ncu full captures of
# the d=128 chain, the d=256 chain and the TMA embed (+ raw / source exports)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], d["roofline_d256"]["roofline"]["frac"], d["roofline_d256"]["value"], d["clocks"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --iters 4 --no-converge --no-extras > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_chain_tc2<" -s 4 -c 1 -o gpurun_out/prof_chain -f python tools/d_probe.py 1 2 > gpurun_out/ncu_chain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2w -s 4 -c 1 -o gpurun_out/prof_chain256 -f python tools/d_probe.py 1 2 > gpurun_out/ncu_chain256.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_embed_tc -s 4 -c 1 -o gpurun_out/prof_embed -f python tools/d_probe.py 1 2 > gpurun_out/ncu_embed.log 2>&1
for r in prof_chain prof_chain256 prof_embed; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>&1
done
ncu -i gpurun_out/prof_chain256.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_chain256_sass.csv 2>&1
ls -la gpurun_out | tail -20
