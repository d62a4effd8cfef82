python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_algorithm1.py -q 2>&1 | tail -3
for b in 256 1024; do timeout 300 python tools/alg1_throughput.py $b 40; done | tee gpurun_out/alg1.jsonl
