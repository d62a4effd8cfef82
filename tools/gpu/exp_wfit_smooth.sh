# fine-tune the fitted SDNet toward smooth boundaries and measure the MFP fixed-point MAE at 2049^2
mkdir -p gpurun_out/fit
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python tools/fit_sdnet.py --init weights/sdnet_fit_d128.npy --steps 30000 --lr 3e-4 --smooth 0.3 --out gpurun_out/fit/w_s03.npy > gpurun_out/fit/w_s03.log 2>&1; tail -1 gpurun_out/fit/w_s03.log
timeout 600 python tools/fit_sdnet.py --init weights/sdnet_fit_d128.npy --steps 30000 --lr 3e-4 --smooth 0.5 --batch 2048 --out gpurun_out/fit/w_s05.npy > gpurun_out/fit/w_s05.log 2>&1; tail -1 gpurun_out/fit/w_s05.log
for w in weights/sdnet_fit_d128.npy gpurun_out/fit/w_s03.npy gpurun_out/fit/w_s05.npy; do
  echo "== $w"
  timeout 600 python tools/iters_to_mae.py --weights $w --only "sdnet W-fit fp16,sdnet W-fit bf16" --grids 1x1 --max 8000 --chunk 200 2>&1 >/dev/null | cut -c1-200
done
