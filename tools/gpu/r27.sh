python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "exact or sine or communication or distributed or placement or boundary" 2>&1 | tail -2
timeout 900 python bench.py --steps 3 > gpurun_out/b27.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b27.json'));t=d['time_to_converge']['exact_subsolver'];print(round(d['value']/1e6,2), t['ms'], t['iterations'], t['ms_without_final_phase'], t['max_err_vs_discrete_solution'])"
