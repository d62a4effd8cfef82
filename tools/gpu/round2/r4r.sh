# (measured, not taken) scatter cache hints: needs the MFP_SC_LDMODE / MFP_SC_STMODE macros (not in the tree); store hints halve the scatter
mkdir -p gpurun_out
for f in "" "-DMFP_SC_STMODE=1" "-DMFP_SC_STMODE=2" "-DMFP_SC_STMODE=3" "-DMFP_SC_LDMODE=2" ""; do
  MFP_NVCC_EXTRA="$f" python paper_2308_14258_b200/build.py --force > gpurun_out/build_ab.log 2>&1 || { tail gpurun_out/build_ab.log; exit 1; }
  echo "flags: $f"
  for i in 1 2; do timeout 300 python tools/bench_io.py 20 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['gather']['frac'],3), round(d['scatter']['us'],2), round(d['scatter']['frac'],3))"; done
done
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
