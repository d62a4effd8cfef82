# (dropped) d = 128 chain cooperative lone last tile (kernel variant not in the tree): slower, tail unchanged
# previous commit's kernel, parity, slot-cycling stress, per-CTA spans
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1
timeout 120 python tools/share_probe.py 4096 4096 1 2>&1 | grep ms
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_fitted_mfp.py tests/test_gpu_slot_cycling.py tests/test_gpu_gelu_erf_tc.py tests/test_gpu_delta.py -m gpu -x -q 2>&1 | tail -3
MFP_NVCC_EXTRA=-DMFP_TRACE python paper_2308_14258_b200/build.py --force > gpurun_out/build_trace.log 2>&1
timeout 300 python tools/chain_trace.py 2>&1 | tail -2
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
