mkdir -p gpurun_out/fit
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python tools/collect_mfp_boundaries.py --out /tmp/mfp_bank.npy 2>&1 | tail -2
timeout 1500 python tools/fit_sdnet.py --init weights/sdnet_fit_d128.npy --steps 60000 --lr 3e-4 --batch 2048 --bank /tmp/mfp_bank.npy --bank-frac 0.5 --smooth 0.25 --out gpurun_out/fit/w_bank.npy > gpurun_out/fit/w_bank.log 2>&1; tail -1 gpurun_out/fit/w_bank.log | cut -c1-300
timeout 600 python tools/iters_to_mae.py --weights gpurun_out/fit/w_bank.npy --only "sdnet W-fit fp16,sdnet W-fit bf16" --grids 1x1 --max 8000 --chunk 200 2>&1 >/dev/null | cut -c1-200
