python paper_2308_14258_b200/build.py > /dev/null 2>&1
echo base; timeout 300 python tools/bench_io.py 10 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['scatter']['us'], d['scatter']['frac'])"
MFP_NVCC_EXTRA="-DMFP_SCATTER_STCS" python paper_2308_14258_b200/build.py --force > /dev/null 2>&1 || MFP_NVCC_EXTRA="-DMFP_SCATTER_STCS" python -c "import sys; sys.path.insert(0,'paper_2308_14258_b200'); import build; build.build(force=True)"
echo stcs; timeout 300 python tools/bench_io.py 10 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['scatter']['us'], d['scatter']['frac'])"
