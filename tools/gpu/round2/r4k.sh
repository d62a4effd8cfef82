# exact subsolver phase kernel with PDL (H_c^T loaded under the predecessor's tail): A/B vs MFP_NO_PDL, parity
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in 0 1 0; do echo "MFP_NO_PDL=$v"; MFP_NO_PDL=$v timeout 120 python tools/exact_probe.py 4096 4096 1024; MFP_NO_PDL=$v timeout 120 python tools/exact_probe.py 1024 2048 1024; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_delta.py tests/test_gpu_device_loop.py tests/test_gpu_persistent.py -m gpu -q -x -k "exact or delta or loop or persist" 2>&1 | tail -2
