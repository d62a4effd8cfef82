mkdir -p gpurun_out/fit
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 300 python training/algorithm1.py --steps 300 --batch 256 2>&1 | tail -1 | cut -c1-300
timeout 300 python training/algorithm1.py --steps 300 --batch 1024 2>&1 | tail -1 | cut -c1-300
timeout 1800 python training/algorithm1.py --init weights/candidates/sdnet_fit_d128_smooth_a.npy --steps 20000 --batch 512 --lr 2e-4 --pde-weight 1e-3 --out gpurun_out/fit/w_pde.npy > gpurun_out/fit/w_pde.log 2>&1; tail -1 gpurun_out/fit/w_pde.log | cut -c1-300; grep "^step" gpurun_out/fit/w_pde.log | tail -3
timeout 600 python tools/iters_to_mae.py --weights gpurun_out/fit/w_pde.npy --only "sdnet W-fit fp16,sdnet W-fit bf16" --grids 1x1 --max 8000 --chunk 200 2>&1 >/dev/null | cut -c1-200
