# chain: SM clock over the work span (clock64 / globaltimer per CTA), at C5; also bench-style nvidia-smi sampling
mkdir -p gpurun_out
MFP_NVCC_EXTRA=-DMFP_TRACE python paper_2308_14258_b200/build.py --force > gpurun_out/build_trace.log 2>&1 || { tail gpurun_out/build_trace.log; exit 1; }
timeout 300 python tools/chain_trace.py
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
nvidia-smi -q -d POWER,CLOCK | grep -E "Power Limit|Current Power|Graphics|SM  " | head -12
(timeout 60 python tools/share_probe.py 4096 4096 2000 > gpurun_out/sp.log 2>&1 &) ; sleep 25; nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv; sleep 2; nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv; wait; cat gpurun_out/sp.log
