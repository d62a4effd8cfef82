mkdir -p gpurun_out
python paper_2308_14258_b200/build.py > /dev/null 2>&1
: > gpurun_out/sanitize_r2.log
sed -n '/^# round-2 host paths/,$p' tools/gpu/round2/sanitize_r2.sh > /tmp/san_tail.sh
bash /tmp/san_tail.sh
