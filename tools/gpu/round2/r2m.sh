python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 300 python tools/bench_io.py 10 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['gather']['us'], d['gather']['frac'], d['scatter']['us'], d['scatter']['frac'])"
timeout 600 python -m pytest tests/test_gpu_boundary_io.py -q 2>&1 | tail -2
