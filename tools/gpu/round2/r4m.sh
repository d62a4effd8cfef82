# exact subsolver: 7 subdomains per warp at C5 (146 blocks on 148 SMs) vs 8 (127 blocks); parity
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in 8 0 8 0; do echo "MFP_EXACT_SUB=$v"; MFP_EXACT_SUB=$v timeout 120 python tools/exact_probe.py 4096 4096 1024; done
timeout 120 python tools/exact_probe.py 2048 4096 1024
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_delta.py tests/test_gpu_device_loop.py tests/test_gpu_persistent.py -m gpu -q -x -k "exact or delta or loop or persist" 2>&1 | tail -2
