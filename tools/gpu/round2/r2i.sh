mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
python -c "import torch; print('reserved smem per block', torch.cuda.get_device_properties(0).reserved_shared_memory_per_block if hasattr(torch.cuda.get_device_properties(0),'reserved_shared_memory_per_block') else 'n/a')"
for u in 8 4; do echo "unroll $u"; MFP_IO_UNROLL=$u timeout 300 python tools/bench_io.py 10 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['gather']['us'], d['gather']['frac'], d['scatter']['us'], d['scatter']['frac'])"; done
timeout 600 python -m pytest tests/test_gpu_boundary_io.py -q 2>&1 | tail -2
export MFP_NO_GRAPHS=1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100000 python -m pytest tests/test_gpu_parity.py -q -x -k "batch_parity and 1000 and 1" > gpurun_out/race_embed_full.log 2>&1
MFP_MAX_PAIRS=2 timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100000 python -m pytest tests/test_gpu_d256.py tests/test_gpu_fp16x.py -q -x -k "(batch_parity and 0-1000-1) or (many_tiles and 333)" > gpurun_out/race_tc_full.log 2>&1
for f in race_embed_full race_tc_full; do echo "== $f"; grep -oE "hazard detected \([^)]*\) at __shared__ 0x[0-9a-f]+" gpurun_out/$f.log | awk '{print $NF}' | sort | uniq -c | sort -k2 | head -20; grep -c "hazard detected" gpurun_out/$f.log; grep -oE "Read Thread.*at [^+]*" gpurun_out/$f.log | sed 's/Read Thread ([0-9,]*) at //' | sort | uniq -c | head; done
