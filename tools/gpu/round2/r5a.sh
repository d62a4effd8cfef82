# (not taken) A/B: split-layer z prefetch depth 1 / 2 / 3 blocks (needs the MFP_SPLIT_PF variant): 1 is best (0.158 vs 0.160 / 0.174 ms)
mkdir -p gpurun_out
for v in pf1 pf2 pf3 pf1 pf2; do
  cp ab/libmfp_$v.so paper_2308_14258_b200/libmfp.so
  echo "lib $v"; timeout 300 python tools/d_probe.py 1 4 2>&1 | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['chain_ms_per_launch'],4), round(d['ms_per_iter'],4))"
done
cp ab/libmfp_pf1.so paper_2308_14258_b200/libmfp.so
