# scatter variants (MFP_SCATTER_V 0..7): one-wave grids, anchor prefetch, U = 2 / 4 / 8, flat per-cell
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
for v in 0 1 2 3 4 5 6 7; do echo -n "v$v "; MFP_SCATTER_V=$v timeout 300 python tools/bench_io.py 20 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['gather']['frac'], round(d['scatter']['us'],2), round(d['scatter']['frac'],3))"; done
for v in 0 2 4 6 7; do MFP_SCATTER_V=$v timeout 600 python -m pytest tests/test_gpu_boundary_io.py -q 2>&1 | tail -1; done
