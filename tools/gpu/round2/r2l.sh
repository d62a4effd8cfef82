python paper_2308_14258_b200/build.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_scatter_phase|k_gather_phase" -s 2 -c 2 -o gpurun_out/prof_io -f python tools/bench_io.py 1 > gpurun_out/ncu_io.log 2>&1
ncu -i gpurun_out/prof_io.ncu-rep --page raw --csv > gpurun_out/prof_io_raw.csv 2>&1
python profiles/summarize.py gpurun_out/prof_io.ncu-rep 2>&1 | head -60
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/prof_io_raw.csv")))
hdr=rows[0]
for v in rows[2:]:
    print(v[hdr.index("Kernel Name")][:40])
    for k in hdr:
        if ("warp_issue_stalled" in k and k.endswith("per_issue_active.ratio")) or k in ("lts__t_sector_hit_rate.pct","dram__throughput.avg.pct_of_peak_sustained_elapsed","sm__warps_active.avg.pct_of_peak_sustained_active","launch__occupancy_limit_registers","launch__registers_per_thread","lts__t_sectors_srcunit_tex_op_write.sum","lts__t_sectors_srcunit_tex_op_read.sum"):
            try:
                if float(v[hdr.index(k)])>0.2: print("  ",k,v[hdr.index(k)])
            except: pass
PY
