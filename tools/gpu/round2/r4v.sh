# (dropped) A/B: d = 128 chain with 3 tile slots x 8 epilogue warps (tc3, not in the tree): 0.174 vs 0.160 ms
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for v in 0 1 0 1; do
  echo "MFP_CHAIN3=$v"; MFP_CHAIN3=$v timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['chain_ms_per_launch'],4), round(d['ms_per_iter'],4))"
  MFP_CHAIN3=$v timeout 120 python tools/share_probe.py 4096 4096 1 2>&1 | grep ms; MFP_CHAIN3=$v timeout 120 python tools/share_probe.py 1024 2048 1 2>&1 | grep ms
done
MFP_CHAIN3=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -m gpu -x -q 2>&1 | tail -3
