# embed v2 (channel-pair conv, no operand MOVs, rows multiple of 16): TC-path parity tests, d_probe, shares, ncu of the embed
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_d256.py tests/test_gpu_fp16x.py tests/test_gpu_bench_parity.py tests/test_gpu_boundary_io.py tests/test_gpu_fitted_mfp.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/d_probe.py 1 4
for s in "4096 4096" "2048 4096" "2048 2048" "1024 2048"; do timeout 120 python tools/share_probe.py $s 1 2>&1 | grep ms; MFP_PROBE_D=256 timeout 120 python tools/share_probe.py $s 1 2>&1 | grep ms; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_embed_tc -s 4 -c 1 -o gpurun_out/prof_embed2 -f python tools/d_probe.py 1 2 > gpurun_out/ncu_embed2.log 2>&1
ncu -i gpurun_out/prof_embed2.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_embed2_sass.csv 2>&1
ncu -i gpurun_out/prof_embed2.ncu-rep --page details --csv > gpurun_out/prof_embed2_details.csv 2>&1
ncu -i gpurun_out/prof_embed2.ncu-rep --page raw --csv > gpurun_out/prof_embed2_raw.csv 2>&1
