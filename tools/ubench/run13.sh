MFP_NVCC_EXTRA="-DMFP_TRACE -DMFP_EXPERIMENT_NO_ACT" python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 300 python tools/chain_trace.py > gpurun_out/trace_noact.txt 2>&1; head -12 gpurun_out/trace_noact.txt
python paper_2308_14258_b200/build.py --force >> gpurun_out/build.log 2>&1
