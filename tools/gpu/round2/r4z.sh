# (not taken) A/B: 32-bit row divisions in the d = 256 and FP16X chains: no gain (0.3466 vs 0.3457, 0.2492 vs 0.2482 ms)
mkdir -p gpurun_out
cp paper_2308_14258_b200/libmfp.so ab/libmfp_new.so
for v in new base new base; do
  cp ab/libmfp_$v.so paper_2308_14258_b200/libmfp.so
  echo "lib $v"; timeout 300 python tools/d_probe.py 1 4 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('d256', round(d['chain_ms_per_launch'],4))"
  timeout 300 python tools/d_probe.py 3 4 2>&1 | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('fp16x', round(d['chain_ms_per_launch'],4))"
done
cp ab/libmfp_new.so paper_2308_14258_b200/libmfp.so
timeout 900 python -m pytest tests/test_gpu_d256.py tests/test_gpu_fp16x.py tests/test_gpu_slot_cycling.py -m gpu -x -q 2>&1 | tail -2
