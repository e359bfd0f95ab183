set -x
python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gram|k_bsr3_spmv_pcg|k_pcg_update|k_pcg_direction|k_gemm_nn" -c 12 -o gpurun_out/prof_r01c python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_ncu.log 2>&1
python bench.py --workload c2 --systems 1 --warmup 0 --steps 1 --no-cpu --no-e2e > gpurun_out/c2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sell1_spmv_pcg" -s 20 -c 2 -o gpurun_out/prof_c2_sell1 python bench.py --workload c2 --systems 1 --warmup 0 --steps 1 --no-cpu --no-e2e > gpurun_out/prof_c2.log 2>&1
python bench.py --systems 2 --warmup 1 --steps 1 --no-cpu --no-e2e > gpurun_out/c3_2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c3_systems2.csv python bench.py --systems 2 --warmup 1 --steps 1 --no-cpu --no-e2e > gpurun_out/launch_ncu.log 2>&1
ls -la gpurun_out/
