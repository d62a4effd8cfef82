python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_p2p_put.py tests/test_gpu_p2p.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 900 python tools/p2p_vs_copy.py --out gpurun_out/p2p_put_vs_copy.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/p2p_put_vs_copy.json')); print({k:(round(v['ms_per_iter_median'],4), round(v['halo_ms_per_iter_profiled'],4)) for k,v in d['transports'].items()}, d['bit_identical'])"
