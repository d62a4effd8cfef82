# A/B in one call: 32-bit row division in the d = 128 chain (current tree) vs the previous build (ab/libmfp_base.so)
mkdir -p gpurun_out
cp paper_2308_14258_b200/libmfp.so ab/libmfp_new.so
for v in new base new base; do
  cp ab/libmfp_$v.so paper_2308_14258_b200/libmfp.so
  echo "lib $v"; timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['chain_ms_per_launch'],4), round(d['ms_per_iter'],4))"
  timeout 120 python tools/share_probe.py 4096 4096 1 2>&1 | grep ms
done
cp ab/libmfp_new.so paper_2308_14258_b200/libmfp.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_slot_cycling.py -m gpu -x -q 2>&1 | tail -2
