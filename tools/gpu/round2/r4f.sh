# A/B: one MMA-issuer warp per tile slot (MFP_MULTI_ISSUER, 20 warps) vs the single in-order issuer
mkdir -p gpurun_out
for f in "" "-DMFP_MULTI_ISSUER" "" "-DMFP_MULTI_ISSUER"; do
  MFP_NVCC_EXTRA="$f" python paper_2308_14258_b200/build.py --force > gpurun_out/build_ab.log 2>&1 || { tail gpurun_out/build_ab.log; exit 1; }
  echo "flags: $f"; timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['chain_ms_per_launch'],4), round(d['ms_per_iter'],4))"
  timeout 120 python tools/share_probe.py 4096 4096 1 2>&1 | grep ms; timeout 120 python tools/share_probe.py 1024 2048 1 2>&1 | grep ms
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -m gpu -x -q 2>&1 | tail -2
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
