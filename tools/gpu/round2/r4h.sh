# A/B (dropped, default 16 best): embed rows per CTA at small batches at the 8-GPU share (needs the MFP_EMBED_MINROWS hack, not in the tree)
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
for r in 0 32 48 0 32; do
  echo "minrows $r"; MFP_EMBED_MINROWS=$r timeout 120 python tools/share_probe.py 1024 2048 1 2>&1 | grep ms; MFP_EMBED_MINROWS=$r timeout 120 python tools/share_probe.py 2048 2048 1 2>&1 | grep ms
done
