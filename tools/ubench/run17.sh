for v in "" "-DMFP_WAIT_NS=32" "-DMFP_WAIT_NS=100" "-DMFP_WAIT_NS=250"; do
MFP_NVCC_EXTRA="$v" python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 300 python bench.py --no-converge --steps 3 > gpurun_out/bench_x.json 2>> gpurun_out/bench.err
python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_x.json').read().strip().splitlines()[-1]); print('variant [$v]', round(d['value']/1e6,2), d['roofline']['chain_ms_per_launch'])"
done
python paper_2308_14258_b200/build.py --force >> gpurun_out/build.log 2>&1
