# d = 256 chain (tc2w): z double-buffered behind an mbarrier, split layer with constant-bank W2 + pipelined z
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_d256.py tests/test_gpu_parity.py tests/test_gpu_fp16x.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/d_probe.py 1 4 2>&1
for s in "4096 4096" "1024 2048"; do MFP_PROBE_D=256 timeout 120 python tools/share_probe.py $s 1 2>&1 | grep ms; done
