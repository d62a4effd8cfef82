MFP_NVCC_EXTRA="-DMFP_EXPERIMENT_NO_ACT -DMFP_EXPERIMENT_NO_MMA -DMFP_EXPERIMENT_NO_TMEM_LD -DMFP_EXPERIMENT_NO_STS" python paper_2308_14258_b200/build.py --force > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2 -s 4 -c 1 -o gpurun_out/prof_skel -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_skel.log 2>&1; tail -1 gpurun_out/ncu_skel.log
python paper_2308_14258_b200/build.py --force >> gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tc2 -s 4 -c 1 -o gpurun_out/prof_chain5 -f python bench.py --steps 1 --warmup 1 --iters 2 --no-converge > gpurun_out/ncu_chain.log 2>&1; tail -1 gpurun_out/ncu_chain.log
