#!/bin/bash
# round-2 kernels under compute-sanitizer: the d = 256 chain (TMA weight ring,
# relay, multicast empty commits), the FP16X split chain, the TMA-staged embed.
# MFP_MAX_PAIRS=2 caps the persistent grids so every ring stage / tile slot
# cycles through many rounds; graphs off so every kernel is a plain launch.
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > /dev/null 2>&1
export MFP_NO_GRAPHS=1
{
for t in memcheck racecheck synccheck; do
  echo "== $t d256 batch"
  MFP_MAX_PAIRS=2 timeout 1200 compute-sanitizer --tool $t --print-limit 10 python -m pytest tests/test_gpu_d256.py -q -x \
    -k "batch_parity and ((0-1000) or (1-37)) and (1 or 2)" 2>&1 | tail -3
  echo "== $t fp16x batch"
  MFP_MAX_PAIRS=2 timeout 1200 compute-sanitizer --tool $t --print-limit 10 python -m pytest tests/test_gpu_fp16x.py -q -x \
    -k "many_tiles and 333" 2>&1 | tail -3
  echo "== $t embed (bf16 batch + field, TMA staging)"
  timeout 1200 compute-sanitizer --tool $t --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "(batch_parity and 1000 and 1) or (tensorcore_field_parity and 64 and 1)" 2>&1 | tail -3
done
echo "== memcheck d256 field + fp16x fitted field"
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_d256.py tests/test_gpu_fp16x.py -q -x \
  -k "(field_parity and 64) or (fitted_field and 128 and sdnet_fit_d128.npy)" 2>&1 | tail -3
} > gpurun_out/sanitize_r2.log 2>&1
cat gpurun_out/sanitize_r2.log
# round-2 host paths: the put transport (epilogue puts, publish / unpack spin
# protocol) and the on-device convergence loop (graphs on: the WHILE node)
{
for t in memcheck synccheck racecheck; do
  echo "== $t p2p put"
  MFP_NO_GRAPHS=1 timeout 900 compute-sanitizer --tool $t --print-limit 10 python -m pytest tests/test_gpu_p2p_put.py -q -x \
    -k "bit_identical and (grid0 or grid2)" 2>&1 | tail -3
done
echo "== memcheck device loop"
unset MFP_NO_GRAPHS
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_device_loop.py -q -x 2>&1 | tail -3
} >> gpurun_out/sanitize_r2.log 2>&1
tail -16 gpurun_out/sanitize_r2.log
