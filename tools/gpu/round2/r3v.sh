# A/B: part of the GELU pairs on an FMA-pipe polynomial (MFP_POLY_EVERY) in the current d = 128 chain
mkdir -p gpurun_out
for f in "" "-DMFP_POLY_EVERY=8" "-DMFP_POLY_EVERY=4" "-DMFP_POLY_EVERY=2"; do
  MFP_NVCC_EXTRA="$f" python paper_2308_14258_b200/build.py --force > gpurun_out/build_ab.log 2>&1 || { tail gpurun_out/build_ab.log; exit 1; }
  echo "flags: $f"; timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1
done
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
