# tc5 (MFP_CHAIN5=1) hang-safe check: a short batch parity run first, then tests and A/B bench
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
MFP_CHAIN5=1 timeout 60 python -m pytest tests/test_gpu_parity.py -q -x -k "batch" > gpurun_out/tc5_quick.log 2>&1
rc=$?; tail -3 gpurun_out/tc5_quick.log; echo "quick rc=$rc"
if [ $rc -eq 0 ]; then
  bash tools/gpu/scripts_gpu_ab.sh MFP_CHAIN5=1 MFP_CHAIN5=0
fi
