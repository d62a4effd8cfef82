python paper_2308_14258_b200/build.py > /dev/null 2>&1
MFP_NO_GRAPHS=1 timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100000 python -m pytest tests/test_gpu_p2p_put.py -q -x -k "bit_identical and (grid0 or grid2)" > gpurun_out/race_put_full.log 2>&1
grep -oE "hazard detected \([^)]*\) at __shared__ 0x[0-9a-f]+" gpurun_out/race_put_full.log | awk '{print $NF}' | sort | uniq -c | sort -k2 | head -20
grep -c "hazard detected" gpurun_out/race_put_full.log
grep -oE "Read Thread.*at [^(]*" gpurun_out/race_put_full.log | sed 's/Read Thread ([0-9,]*) (block rank [0-9]*) at //' | sort | uniq -c | head
