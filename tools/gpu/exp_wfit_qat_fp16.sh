# does a short fp16-QAT pass make the bf16-aware fit robust in fp16 as well?
mkdir -p gpurun_out/fit
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python tools/collect_mfp_boundaries.py --out /tmp/mfp_bank.npy 2>&1 | tail -1
timeout 1500 python tools/fit_sdnet.py --init weights/sdnet_fit_d128_mfp.npy --steps 20000 --lr 1e-4 --batch 2048 --bank /tmp/mfp_bank.npy --bank-frac 0.5 --smooth 0.25 --qat fp16 --seed 7 --out gpurun_out/fit/w_qat16.npy > gpurun_out/fit/w_qat16.log 2>&1; tail -1 gpurun_out/fit/w_qat16.log | cut -c1-200
timeout 900 python tools/iters_to_mae.py --weights gpurun_out/fit/w_qat16.npy --only "sdnet W-fit fp16,sdnet W-fit bf16" --grids 1x1 --max 8000 --chunk 100 2>&1 >/dev/null | cut -c1-200
timeout 1500 python tools/iters_to_mae.py --n 4096 --weights gpurun_out/fit/w_qat16.npy --only "sdnet W-fit bf16,sdnet W-fit fp16" --grids 1x1 --max 20000 --chunk 200 2>&1 >/dev/null | cut -c1-200
