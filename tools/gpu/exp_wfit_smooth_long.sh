# longer smooth-boundary fits of the SDNet; MFP fixed-point MAE at 2049^2 for each
mkdir -p gpurun_out/fit
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 1500 python tools/fit_sdnet.py --init weights/candidates/sdnet_fit_d128_s05.npy --steps 100000 --lr 2e-4 --smooth 0.5 --batch 2048 --out gpurun_out/fit/w_a.npy > gpurun_out/fit/w_a.log 2>&1; tail -1 gpurun_out/fit/w_a.log | cut -c1-300
timeout 1500 python tools/fit_sdnet.py --steps 120000 --lr 1e-3 --smooth 0.4 --batch 2048 --seed 1 --out gpurun_out/fit/w_b.npy > gpurun_out/fit/w_b.log 2>&1; tail -1 gpurun_out/fit/w_b.log | cut -c1-300
for w in gpurun_out/fit/w_a.npy gpurun_out/fit/w_b.npy; do
  echo "== $w"
  timeout 600 python tools/iters_to_mae.py --weights $w --only "sdnet W-fit fp16,sdnet W-fit bf16" --grids 1x1 --max 8000 --chunk 200 2>&1 >/dev/null | cut -c1-200
done
