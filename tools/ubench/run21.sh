nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include -o /tmp/act tools/ubench/act.cu && /tmp/act > gpurun_out/act.txt 2>&1; cat gpurun_out/act.txt
