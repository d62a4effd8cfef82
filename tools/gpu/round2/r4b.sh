# FP16X chain (tc2s): z double-buffered behind an mbarrier, split layer with constant-bank W2 + pipelined z
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_fp16x.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/d_probe.py 3 4 2>&1 | head -1
timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1
