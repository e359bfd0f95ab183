# ncu --set full of the SpMV kernels after the scipy-exact row sums (row_madd)
python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bsr3_spmv_pcg" -s 70 -c 2 -o gpurun_out/prof_spmv_e python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_spmv_e.log 2>&1
python bench.py --workload c2 --systems 1 --warmup 0 --steps 1 --no-cpu --no-e2e > gpurun_out/c2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sell1_spmv_pcg" -s 20 -c 2 -o gpurun_out/prof_sell1_e python bench.py --workload c2 --systems 1 --warmup 0 --steps 1 --no-cpu --no-e2e > gpurun_out/prof_sell1_e.log 2>&1
