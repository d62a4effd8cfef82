# d = 128 chain: fresh clock64 timeline (MFP_TRACE build) + ncu full capture with source of the committed kernel
mkdir -p gpurun_out
MFP_NVCC_EXTRA=-DMFP_TRACE python paper_2308_14258_b200/build.py --force > gpurun_out/build_trace.log 2>&1 || { tail gpurun_out/build_trace.log; exit 1; }
timeout 300 python tools/chain_trace.py
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_chain_tc2$" -s 4 -c 1 -o gpurun_out/prof_chain3 -f python tools/d_probe.py 1 2 > gpurun_out/ncu_chain3.log 2>&1
ncu -i gpurun_out/prof_chain3.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_chain3_sass.csv 2>&1
ncu -i gpurun_out/prof_chain3.ncu-rep --page raw --csv > gpurun_out/prof_chain3_raw.csv 2>&1
ncu -i gpurun_out/prof_chain3.ncu-rep --page details --csv > gpurun_out/prof_chain3_details.csv 2>&1
ls -la gpurun_out/prof_chain3*
