# product scatter (U = 2, 8 blocks / SM, one wave, fused last-block reduction): tests + bench_io
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_boundary_io.py -q 2>&1 | tail -3
for i in 1 2; do timeout 300 python tools/bench_io.py 20 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['gather']['frac'],3), round(d['scatter']['us'],2), round(d['scatter']['frac'],3))"; done
