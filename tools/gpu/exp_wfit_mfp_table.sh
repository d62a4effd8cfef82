# the paper's Table strongScalingIter analog with the MFP-distribution fitted weights (fp16),
# at 2049^2 (the paper's domain) and 4097^2 (C5), processor grids emulated on one GPU
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 1200 python tools/iters_to_mae.py --weights weights/sdnet_fit_d128_mfp.npy --only "sdnet W-fit fp16" --grids 1x1,1x2,2x2,2x4 --max 12000 --chunk 100 > gpurun_out/iters_mfp_2049.json 2> gpurun_out/iters_mfp_2049.err; cut -c1-220 gpurun_out/iters_mfp_2049.err
timeout 1500 python tools/iters_to_mae.py --n 4096 --weights weights/sdnet_fit_d128_mfp.npy --only "sdnet W-fit fp16,exact fp32" --grids 1x1 --max 30000 --chunk 200 > gpurun_out/iters_mfp_4097.json 2> gpurun_out/iters_mfp_4097.err; cut -c1-220 gpurun_out/iters_mfp_4097.err
