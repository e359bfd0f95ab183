# Round-2 measurement job: the -m gpu suite, then every bench line kept under profiles/ (one B200).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/r02_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err; echo c3_rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo ref_rc=$?
timeout 600 python bench.py --workload c1 > gpurun_out/r02_bench_c1.json 2> gpurun_out/r02_bench_c1.err; echo c1_rc=$?
timeout 900 python bench.py --workload c2 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err; echo c2_rc=$?
timeout 900 python bench.py --workload c5 > gpurun_out/r02_bench_c5_m2048.json 2> gpurun_out/r02_bench_c5_m2048.err; echo c5_rc=$?
timeout 900 python bench.py --workload c5 --m 256 > gpurun_out/r02_bench_c5_m256.json 2> gpurun_out/r02_bench_c5_m256.err; echo c5b_rc=$?
timeout 1500 python bench.py --mode fom --warmup 1 --no-cpu > gpurun_out/r02_bench_c3_fom.json 2> gpurun_out/r02_bench_c3_fom.err; echo fom_rc=$?
timeout 2400 python bench.py --workload c4 --warmup 1 --no-cpu > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo c4_rc=$?
