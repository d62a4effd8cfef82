mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
for s in "1024 2048" "2048 2048" "2048 4096" "4096 4096"; do timeout 120 python tools/share_probe.py $s; done > gpurun_out/share.txt 2>&1
for s in "1024 2048" "2048 2048"; do MFP_EMBED_SIMT=1 timeout 120 python tools/share_probe.py $s; done >> gpurun_out/share.txt 2>&1
for s in "1024 2048" "2048 2048"; do MFP_NO_PDL=1 timeout 120 python tools/share_probe.py $s; done >> gpurun_out/share.txt 2>&1
cat gpurun_out/share.txt
