# d = 128 chain weights by TMA bulk copies (waited after the PDL wait): parity + timing + per-CTA spans
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_fitted_mfp.py tests/test_gpu_delta.py tests/test_gpu_device_loop.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1
for s in "4096 4096" "1024 2048"; do timeout 120 python tools/share_probe.py $s 1 2>&1 | grep ms; done
MFP_NVCC_EXTRA=-DMFP_TRACE python paper_2308_14258_b200/build.py --force > gpurun_out/build_trace.log 2>&1
timeout 300 python tools/chain_trace.py
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
