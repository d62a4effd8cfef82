# (dropped) A/B: degree-7 FMA-pipe GELU on 1 of N pairs (needs the r4p gelu2_poly variant, not in the tree): no gain
mkdir -p gpurun_out
for f in "" "-DMFP_POLY_EVERY=4" "-DMFP_POLY_EVERY=3" "-DMFP_POLY_EVERY=8" "" "-DMFP_POLY_EVERY=4"; do
  MFP_NVCC_EXTRA="$f" python paper_2308_14258_b200/build.py --force > gpurun_out/build_ab.log 2>&1 || { tail gpurun_out/build_ab.log; exit 1; }
  echo "flags: $f"; timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['chain_ms_per_launch'],4), round(d['ms_per_iter'],4))"
  timeout 120 python tools/share_probe.py 4096 4096 1 2>&1 | grep ms
done
MFP_NVCC_EXTRA="-DMFP_POLY_EVERY=4" python paper_2308_14258_b200/build.py --force > gpurun_out/build_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_fitted_mfp.py tests/test_gpu_gelu_erf_tc.py -m gpu -q 2>&1 | tail -3
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
