mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
for v in 0 1; do for s in "1024 2048" "2048 2048" "4096 4096"; do echo -n "2slot=$v "; MFP_CHAIN_2SLOT=$v timeout 120 python tools/share_probe.py $s; done; done > gpurun_out/share2.txt 2>&1
cat gpurun_out/share2.txt
MFP_CHAIN_2SLOT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "tensorcore or batch" > gpurun_out/t2slot.log 2>&1; tail -3 gpurun_out/t2slot.log
