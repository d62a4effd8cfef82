# the QAT (bf16) MFP-distribution fit: MAE trajectory past the bar, grids, and C5
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
W=weights/candidates/sdnet_fit_d128_qat.npy
timeout 900 python tools/iters_to_mae.py --weights $W --only "sdnet W-fit fp16,sdnet W-fit bf16" --grids 1x1 --max 6000 --chunk 100 --target 0.0 > gpurun_out/qat_traj_2049.json 2> /dev/null
python -c "
import json; d=json.load(open('gpurun_out/qat_traj_2049.json'))
for r in d['rows']: print(r['subsolver'], [(a, round(b,4)) for a,b in r['mae_history']])"
timeout 900 python tools/iters_to_mae.py --weights $W --only "sdnet W-fit bf16,sdnet W-fit fp16" --grids 1x1,1x2,2x2,2x4 --max 8000 --chunk 50 > gpurun_out/qat_grids_2049.json 2> gpurun_out/qat_grids.err; cut -c1-200 gpurun_out/qat_grids.err
timeout 1500 python tools/iters_to_mae.py --n 4096 --weights $W --only "sdnet W-fit bf16,sdnet W-fit fp16" --grids 1x1 --max 30000 --chunk 200 > gpurun_out/qat_4097.json 2> gpurun_out/qat_4097.err; cut -c1-200 gpurun_out/qat_4097.err
