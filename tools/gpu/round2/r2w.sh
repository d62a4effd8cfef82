python paper_2308_14258_b200/build.py > /dev/null 2>&1
for v in 0 1; do for s in "1024 2048" "2048 2048" "4096 4096"; do echo -n "half=$v "; MFP_CHAIN_HALF=$v timeout 120 python tools/share_probe.py $s; done; done 2>&1
MFP_CHAIN_HALF=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "tensorcore or batch" 2>&1 | tail -2
