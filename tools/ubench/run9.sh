MFP_NVCC_EXTRA="-DMFP_TRACE" python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 300 python tools/chain_trace.py > gpurun_out/trace.txt 2>&1; cat gpurun_out/trace.txt | head -40
MFP_L0_SIMT=1 timeout 300 python tools/chain_trace.py > gpurun_out/trace_simt.txt 2>&1; head -14 gpurun_out/trace_simt.txt
