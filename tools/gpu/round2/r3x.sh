# chain per-CTA globaltimer spans (MFP_TRACE build): prologue, work span, tail
mkdir -p gpurun_out
MFP_NVCC_EXTRA=-DMFP_TRACE python paper_2308_14258_b200/build.py --force > gpurun_out/build_trace.log 2>&1 || { tail gpurun_out/build_trace.log; exit 1; }
timeout 300 python tools/chain_trace.py
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
