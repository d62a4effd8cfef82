# scatter variants round 2: U2/8 (+prefetch), U4/6, U3/6 prefetch, fused last-block reduction (11-13)
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
for v in 5 8 9 10 11 12 13 5 11 13; do echo -n "v$v "; MFP_SCATTER_V=$v timeout 300 python tools/bench_io.py 20 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['scatter']['us'],2), round(d['scatter']['frac'],3))"; done
for v in 11 12 13; do MFP_SCATTER_V=$v timeout 600 python -m pytest tests/test_gpu_boundary_io.py -q 2>&1 | tail -1; done
