# second MFP-distribution round: boundaries from 4097^2 exact runs, continue from the 2049^2 fit
mkdir -p gpurun_out/fit
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python tools/collect_mfp_boundaries.py --n 4096 --seeds 3 --at 0,4,16,64,256,1024,2048,4096 --per 5000 --out /tmp/mfp_bank_c5.npy 2>&1 | tail -1
timeout 600 python tools/collect_mfp_boundaries.py --n 2048 --seeds 2 --per 4000 --out /tmp/mfp_bank_c3.npy 2>&1 | tail -1
python -c "import numpy as np; np.save('/tmp/mfp_bank_all.npy', np.concatenate([np.load('/tmp/mfp_bank_c5.npy'), np.load('/tmp/mfp_bank_c3.npy')]))"
timeout 1500 python tools/fit_sdnet.py --init weights/sdnet_fit_d128_mfp.npy --steps 60000 --lr 2e-4 --batch 2048 --bank /tmp/mfp_bank_all.npy --bank-frac 0.6 --smooth 0.2 --seed 3 --out gpurun_out/fit/w_bank2.npy > gpurun_out/fit/w_bank2.log 2>&1; tail -1 gpurun_out/fit/w_bank2.log | cut -c1-300
timeout 600 python tools/iters_to_mae.py --weights gpurun_out/fit/w_bank2.npy --only "sdnet W-fit fp16" --grids 1x1 --max 8000 --chunk 100 2>&1 >/dev/null | cut -c1-200
timeout 1500 python tools/iters_to_mae.py --n 4096 --weights gpurun_out/fit/w_bank2.npy --only "sdnet W-fit fp16" --grids 1x1 --max 30000 --chunk 200 2>&1 >/dev/null | cut -c1-200
