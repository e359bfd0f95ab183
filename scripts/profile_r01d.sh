# targeted ncu --set full captures of the C3 kernels (scripts/profile_kernels.py workload)
python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gram" -c 3 -o gpurun_out/prof_gram python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_gram.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_update|k_pcg_direction" -s 124 -c 4 -o gpurun_out/prof_stage3 python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_stage3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_nn" -c 1 -o gpurun_out/prof_gemm python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_gemm.log 2>&1
ls -la gpurun_out/
