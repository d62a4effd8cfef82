# chain per-CTA spans at the 8-GPU share's phase size (B ~ 2,050) and at C5; embed timing at small batch
mkdir -p gpurun_out
MFP_NVCC_EXTRA=-DMFP_TRACE python paper_2308_14258_b200/build.py --force > gpurun_out/build_trace.log 2>&1 || { tail gpurun_out/build_trace.log; exit 1; }
for b in 2048 4096 16256; do echo "B=$b"; MFP_TRACE_B=$b timeout 300 python tools/chain_trace.py 2>&1 | tail -3; done
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_share.csv python tools/share_probe.py 1024 2048 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_share.csv")))
h = [r for r in rows if r and r[0] == "ID"][0]
i_k, i_v = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[rows.index(h) + 1:]:
    if len(r) > i_v: d[r[i_k][:40]].append(float(r[i_v]))
for k, v in d.items(): print(f"{k:40s} n={len(v):4d} median_us={sorted(v)[len(v)//2]/1e3:.2f}")
PY
