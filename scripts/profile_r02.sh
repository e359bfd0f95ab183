# r02 evidence: ncu --set full of the TMA-staged Gram and the fused PCG vector kernels, launch list of a 2-system bench
set -x
python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_gram_tma" -c 3 -o gpurun_out/prof_r02_gram python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_r02_gram.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_update|k_pcg_direction" -s 140 -c 4 -o gpurun_out/prof_r02_stage3 python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_r02_stage3.log 2>&1
python bench.py --systems 2 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_systems2_plain_r02.json 2> gpurun_out/bench_systems2_plain_r02.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_systems2_r02.csv python bench.py --systems 2 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_systems2_ncu_r02.log 2>&1
python scripts/e2e_probe.py 40 > gpurun_out/r02h_e2e_probe.json 2> gpurun_out/r02h_e2e_probe.err
cat gpurun_out/r02h_e2e_probe.json
ls -la gpurun_out/*.ncu-rep
# the SpMV kernel with the same build (the bench line's `traffic`)
ncu --set full --clock-control none --import-source on -k regex:"k_bsr3_spmv_pcg" -s 70 -c 2 -o gpurun_out/prof_r02_spmv python scripts/profile_kernels.py --iters 12 > gpurun_out/prof_r02_spmv.log 2>&1
