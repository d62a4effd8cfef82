python paper_2308_14258_b200/build.py > gpurun_out/build.log 2>&1
bash tools/gpu/scripts_gpu_ab.sh MFP_X=0 MFP_NO_PDL=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
