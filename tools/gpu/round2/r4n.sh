# exact subsolver k-loop unroll A/B (MFP_EXACT_UNROLL 2 / 4 / 8) at C5 and the 2-GPU share
mkdir -p gpurun_out
for u in 2 4 8 2; do
  MFP_NVCC_EXTRA="-DMFP_EXACT_UNROLL=$u" python paper_2308_14258_b200/build.py --force > gpurun_out/build_ab.log 2>&1 || { tail gpurun_out/build_ab.log; exit 1; }
  echo "unroll $u"; timeout 120 python tools/exact_probe.py 4096 4096 1024; timeout 120 python tools/exact_probe.py 1024 2048 1024
done
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
