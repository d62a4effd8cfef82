mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > /dev/null 2>&1
export MFP_NO_GRAPHS=1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 6 python -m pytest tests/test_gpu_parity.py -q -x -k "batch_parity and 1000 and 1" > gpurun_out/race_embed.log 2>&1
MFP_MAX_PAIRS=2 timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 6 python -m pytest tests/test_gpu_d256.py -q -x -k "batch_parity and 0-1000-1" > gpurun_out/race_d256.log 2>&1
MFP_MAX_PAIRS=2 timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 6 python -m pytest tests/test_gpu_fp16x.py -q -x -k "many_tiles and 333" > gpurun_out/race_fp16x.log 2>&1
for f in race_embed race_d256 race_fp16x; do echo "=== $f"; grep -E "Race|hazard|Write|Read|at 0x|in /|SUMMARY" gpurun_out/$f.log | head -40; done
