# A/B: mbarrier wait variants in the current chains (default try_wait + suspend hint, spin, nanosleep back-off)
mkdir -p gpurun_out
for f in "" "-DMFP_WAIT_NS=64" "-DMFP_WAIT_NS=200" "-DMFP_WAIT_SPIN" ""; do
  MFP_NVCC_EXTRA="$f" python paper_2308_14258_b200/build.py --force > gpurun_out/build_ab.log 2>&1 || { tail gpurun_out/build_ab.log; exit 1; }
  echo "flags: $f"; timeout 300 python tools/d_probe.py 1 4 2>&1 | python -c "import sys,json; [print(json.loads(l)['d'], round(json.loads(l)['chain_ms_per_launch'],4), round(json.loads(l)['ms_per_iter'],4)) for l in sys.stdin]"
done
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
