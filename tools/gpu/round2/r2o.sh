python paper_2308_14258_b200/build.py > /dev/null 2>&1
for d in 128 256; do for s in "4096 4096" "2048 4096" "2048 2048" "1024 2048"; do MFP_PROBE_D=$d timeout 200 python tools/share_probe.py $s; done; done 2>&1 | tee gpurun_out/share_d.txt
