python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_final_lines --csv python tools/d_probe.py 1 1 2>/dev/null | grep k_final_lines | head -3
