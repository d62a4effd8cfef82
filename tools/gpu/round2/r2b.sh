mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
for a in "4096 1 3" "1024 1 3" "4096 2 3" "512 1 3"; do timeout 300 python tools/diag_final.py $a >> gpurun_out/diag_final.jsonl 2>>gpurun_out/diag.err; done
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/gpu_tests.log 2>&1
tail -40 gpurun_out/gpu_tests.log
