python paper_2308_14258_b200/build.py > /dev/null 2>&1
echo "fused ticket (new), read-flush"; timeout 300 python tools/bench_io.py 10 x | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['gather']['us'], d['gather']['frac'], d['scatter']['us'], d['scatter']['frac'])"
cp tools/gpu/_old/kernels_boundary_io.cu paper_2308_14258_b200/csrc/; cp tools/gpu/_old/api.cu paper_2308_14258_b200/csrc/
python paper_2308_14258_b200/build.py > /dev/null 2>&1
echo "old (separate reduce), read-flush"; timeout 300 python tools/bench_io.py 10 x | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['gather']['us'], d['gather']['frac'], d['scatter']['us'], d['scatter']['frac'])"
