#!/bin/bash
# compute-sanitizer over the GPU parity tests (graphs off so every kernel is a plain launch)
python paper_2308_14258_b200/build.py > /dev/null 2>&1
export MFP_NO_GRAPHS=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "batch_parity or phase_placement or exact_fixed_k_parity or full_size_sampled" 2>&1 | tail -4
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_boundary_io.py -q -x -k "not 1024" 2>&1 | tail -4
for t in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -k "batch_parity and 333" 2>&1 | tail -3
done
# many rounds per tile slot: the persistent chain capped at 2 CTA pairs (MFP_MAX_PAIRS),
# B = 1000 -> 239 pair tiles -> ~30 tiles per slot (mbarrier parities, z prefetch and
# the two z copies cycle through many rounds); a 512^2 bf16 / fp16 field likewise
for t in racecheck synccheck; do
  MFP_MAX_PAIRS=2 timeout 1500 compute-sanitizer --tool $t --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "(batch_parity and 1000) or (tensorcore_field_parity and 512)" 2>&1 | tail -3
done
# NEXT-2 peer-memory transport (spin-waits on epoch flags, last-block publication)
for t in memcheck synccheck racecheck; do
  MFP_NO_GRAPHS=1 timeout 900 compute-sanitizer --tool $t --print-limit 10 python -m pytest tests/test_gpu_p2p.py -q -x \
    -k "grid0 or grid3 or errors" 2>&1 | tail -3
done
