python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
bash tools/gpu/scripts_gpu_ab.sh MFP_CHAIN5=1 MFP_CHAIN5=0
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
