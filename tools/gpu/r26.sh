python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do timeout 600 python bench.py --no-converge > gpurun_out/b26.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b26.json'));print(round(d['value']/1e6,2), round(d['e2e']['value']/1e6,2))"; done
