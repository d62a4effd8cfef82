# exact subsolver at C5: launch list (per-kernel durations) + ncu full capture of k_exact_phase (source)
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_exact.csv python tools/exact_probe.py 4096 4096 16 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_exact.csv")))
h = [r for r in rows if r and r[0] == "ID"][0]
i_k, i_v = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[rows.index(h) + 1:]:
    if len(r) > i_v: d[r[i_k][:50]].append(float(r[i_v]))
for k, v in d.items(): print(f"{k:50s} n={len(v):4d} median_us={sorted(v)[len(v)//2]/1e3:.2f}")
PY
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exact_phase -s 8 -c 1 -o gpurun_out/prof_exact -f python tools/exact_probe.py 4096 4096 16 > gpurun_out/ncu_exact.log 2>&1
ncu -i gpurun_out/prof_exact.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_exact_sass.csv 2>&1
ncu -i gpurun_out/prof_exact.ncu-rep --page raw --csv > gpurun_out/prof_exact_raw.csv 2>&1
ncu -i gpurun_out/prof_exact.ncu-rep --page details --csv > gpurun_out/prof_exact_details.csv 2>&1
