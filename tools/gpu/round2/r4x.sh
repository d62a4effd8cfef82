# embed at the 8-GPU share's batch (B ~ 2,050): ncu full capture with source
mkdir -p gpurun_out
python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_embed_tc -s 8 -c 1 -o gpurun_out/prof_embed_share -f python tools/share_probe.py 1024 2048 2 > gpurun_out/ncu_embed_share.log 2>&1
ncu -i gpurun_out/prof_embed_share.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_embed_share_sass.csv 2>&1
ncu -i gpurun_out/prof_embed_share.ncu-rep --page details --csv > gpurun_out/prof_embed_share_details.csv 2>&1
tail -3 gpurun_out/ncu_embed_share.log
